#!/usr/bin/env python
"""Benchmark: CIA Kuramoto RK4 on BASELINE.json configs[1] (config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json:2): node-updates/s = N_nodes x RK4 steps / time, one
node-update = one node advanced by one full RK4 step (4 CIA RHS evaluations).

Timing protocol (ours):
* inputs (graph CSR, theta, omega) resident in HBM before the timed region;
* every timed step is one replay of a captured CUDA graph holding one RK4 step
  (the persistent RK4 kernel: 4 fused stages with grid barriers, + 1
  bookkeeping kernel); L2 (126 MB) is FLUSHED before every step by writing a
  512 MB buffer outside the events, so each step streams its CSR from HBM in
  stage 1 (config 2's inputs, ~60 MB compressed, are smaller than L2);
* CUDA events on the launching stream, barrier + synchronize on both sides,
  max over ranks; value = N x K / sum(step times).
Extra keys: roofline of the timed kernel (4 x canonical RHS bytes per launch
/ measured step time), the CPU baseline (the REAL reference, baseline/_ref
commdyn with its numba kernels as shipped, pinned to one core, bounded
sample), e2e through the public integrate() API with host arrays, clocks
sampled during the run, gpu_launches.

--impl reference runs the unmodified reference (baseline/_ref/commdyn, numba
backend as shipped: single-threaded kernels) through its own public kernel
dispatchers, composed by the SPEC orchestration (oracle/cia.py), on the same
config; if baseline/_ref is absent it falls back to the oracle C port with
all host threads and says so.

--gpus N without WORLD_SIZE in the environment launches N ranks itself
(torch.distributed.run on 127.0.0.1), as the driver does for its scaling run.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "node-updates/sec (CIA Kuramoto RK4 RHS)"
UNIT = "node-updates/s"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic_bytes(kernel: str = "ell_rk4_kernel"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of ``kernel``
    from the committed `ncu --set full` capture of the same build
    (profiles/rNN_<kernel>_ncu_raw.csv, the newest round)."""
    import csv
    import glob

    files = sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_{kernel}_ncu_raw.csv")))
    if not files:
        return None, None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    with open(files[-1]) as f:
        rows = list(csv.reader(f))
    hdr, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(name)
        tot += float(vals[i].replace(",", "")) * scale.get(units[i], 1)
    return tot, os.path.basename(files[-1])


def algorithmic_bytes_per_rhs(n: int, nnz_dir: int, d: int = 1, n_param: int = 1) -> int:
    """B_rhs = 4 nnz_dir + 8 (N+1) + N (16 d + 8 n_param)."""
    return 4 * nnz_dir + 8 * (n + 1) + n * (16 * d + 8 * n_param)


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        util = [float(s[6]) for s in self.samples if s[6].replace(".", "").isdigit()]
        loaded = [c for c, u in zip(sm, util) if u > 0] or sm
        reasons = sorted({n for s in self.samples for n, v in zip(self.NAMES, s[2:6])
                          if v.lower().startswith("active")})
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def load_reference():
    """The unmodified reference package installed under baseline/_ref (pip
    --target).  Returns (commdyn._kernels, backend name) or
    (None, why).  numba's JIT cache goes to a writable temp dir
    (commdyn/_backend.py:61-63 compiles with cache=True)."""
    ref_dir = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref_dir, "commdyn", "_kernels.py")):
        return None, "baseline/_ref/commdyn not installed"
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/commdyn_numba_cache")
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    saved = os.environ.pop("COMMDYN_BACKEND", None)  # reference default: numba if importable
    try:
        from commdyn import _backend as rb, _kernels as rk
    except Exception as e:  # noqa: BLE001
        return None, f"import failed: {e}"
    finally:
        if saved is not None:
            os.environ["COMMDYN_BACKEND"] = saved
    return rk, rb.backend()


def _cpu_rk4_rate(kern, case, dec, omega, theta0, steps: int):
    """``steps`` full RK4 steps of the whole graph through ``kern``'s
    dispatchers (order_params_blocks + dense_complex + pairs_trig), SPEC
    orchestration of oracle/cia.py.  Returns (node-updates/s, seconds)."""
    from oracle import cia

    s = dec.correction

    def rhs(x):
        return cia.kuramoto_rhs_cia(kern, x, omega, dec.offsets, s.iu, s.iv, s.sgn,
                                    case.coupling, case.n)

    t = time.perf_counter()
    cia.rk4_integrate(rhs, theta0, case.dt, steps)
    el = time.perf_counter() - t
    return case.n * steps / el, el


def _warm_reference(kern):
    """Compile the reference's numba kernels on a tiny input (outside timing)."""
    from oracle import cia

    x = np.linspace(-3, 3, 8)
    off = np.array([0, 4, 8], dtype=np.int64)
    iu = np.array([0, 1], dtype=np.int64)
    iv = np.array([1, 5], dtype=np.int64)
    cia.kuramoto_rhs_cia(kern, x, np.zeros(8), off, iu, iv, np.array([-1.0, 1.0]), 1.0, 8)


def cpu_baseline_sample(case, dec, omega, theta0, steps: int = 3):
    """The real reference (baseline/_ref commdyn, numba as shipped) pinned to
    ONE host core (taskset -c 0 equivalent via
    sched_setaffinity), JIT warmed first; falls back to the oracle C port
    (1 thread) when baseline/_ref is absent.  Returns the cpu_baseline dict."""
    kern, backend = load_reference()
    kind = "reference"
    if kern is None:
        from oracle import kernels as kern  # noqa: N813

        kern.set_threads(1)
        kind, backend = "port", f"oracle C port ({backend})"
    else:
        _warm_reference(kern)
    aff = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    try:
        if aff:
            os.sched_setaffinity(0, {min(aff)})
        rate, el = _cpu_rk4_rate(kern, case, dec, omega, theta0, steps)
    finally:
        if aff:
            os.sched_setaffinity(0, aff)
    src = ("baseline/_ref commdyn._kernels (unmodified reference, numba backend, "
           "single-threaded as shipped)" if kind == "reference" else backend)
    return {"value": rate, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{steps} full RK4 steps of config 2 ({el:.1f} s) through {src}, "
                      f"SPEC orchestration (oracle/cia.py), pinned to 1 of {os.cpu_count()} "
                      "host cores"}


def cfg2_config(case, dec):
    """The workload description both arms print (identical dicts)."""
    return {"workload": "cfg2 Kuramoto CIA RK4, SBM N=200000, 200 power-law communities, "
                        "p_in .95, inter degree 5, K=5 (global 1/N), dt .01",
            "n_nodes": case.n, "n_comm": int(len(case.sizes)), "nnz_dir": int(dec.nnz_dir),
            "dt": case.dt, "l2": "GPU arm: L2 flushed (512 MB write) before every timed step"}


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return 0
    from paper_2203_16657_b200 import configs

    case = configs.config2()
    dec = case.decomposition()
    omega, theta0 = case.state()
    kern, backend = load_reference()
    if kern is not None:
        _warm_reference(kern)
        kind, cores = "reference", 1
        src = (f"baseline/_ref commdyn._kernels (unmodified reference, {backend} backend; its "
               "kernels are single-threaded as shipped, _kernels.py:4-6)")
    else:
        from oracle import kernels as kern  # noqa: N813

        cores = max(1, os.cpu_count() or 1)
        kern.set_threads(cores)
        kind = "port"
        src = (f"oracle C port of commdyn/_kernels.py, {cores} OpenMP threads "
               f"(reference unavailable: {backend})")
    W, K = args.warmup, args.steps
    t_w = 0.0
    if W:
        _, t_w = _cpu_rk4_rate(kern, case, dec, omega, theta0, W)
    per_step = t_w / W if W else None
    budget_s = 900.0
    if per_step is None:
        _, per_step = _cpu_rk4_rate(kern, case, dec, omega, theta0, 1)
    steps = int(max(1, min(K, budget_s // max(per_step, 1e-3))))
    rate, el = _cpu_rk4_rate(kern, case, dec, omega, theta0, steps)
    sample = (f"{steps} full RK4 steps of config 2 (N={case.n}, nnz_dir={dec.nnz_dir}) after "
              f"{W} warm-up steps, from theta0; {src}; SPEC orchestration (oracle/cia.py)"
              + ("" if steps == K else f"; bounded to {budget_s:.0f} s of the requested {K}"))
    line = {
        "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": W, "ms_per_step": 1e3 * el / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": cfg2_config(case, dec),
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch

    rank, world, local = _dist_env()
    if world > 1 or os.environ.get("CDK_BENCH_SHARDED") == "1":  # (1-rank: path check)
        from paper_2203_16657_b200 import multi

        return multi.bench_main(args)
    torch.cuda.set_device(local)
    from paper_2203_16657_b200 import _lib, configs
    from paper_2203_16657_b200.engine import KuramotoEngine
    from paper_2203_16657_b200.plan import DeviceGraph

    lib = _lib.lib()
    case = configs.config2()
    t0 = time.perf_counter()
    dec = case.decomposition()
    t_gen = time.perf_counter() - t0
    omega, theta0 = case.state()
    t0 = time.perf_counter()
    dg = DeviceGraph(dec)
    t_plan = time.perf_counter() - t0
    eng = KuramotoEngine(dec, omega, coupling=case.coupling, norm=case.n, graph=dg)
    eng.set_state(theta0)
    n, nnz = case.n, dec.nnz_dir
    dt = case.dt

    stream = torch.cuda.Stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush_l2():
        flush.fill_(float(np.random.random()))

    # capture one RK4 step as a CUDA graph
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        eng.rk4(dt, 1, stream=stream)  # warm + attribute setup outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    lc0 = int(lib.cdk_launch_count())
    with torch.cuda.graph(graph, stream=stream):
        eng.rk4(dt, 1, stream=stream)
    torch.cuda.synchronize()
    per_step_launches = int(lib.cdk_launch_count()) - lc0  # kernels one captured step holds

    W, K = max(3, args.warmup), args.steps
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(W):
            flush_l2()
            graph.replay()
        torch.cuda.synchronize()
        eng.set_state(theta0)  # the timed trajectory starts at theta0
        torch.cuda.synchronize()
        _barrier(world)
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        l0 = int(lib.cdk_launch_count())
        cur = torch.cuda.current_stream()
        for i in range(K):
            flush_l2()
            starts[i].record(cur)
            graph.replay()
            ends[i].record(cur)
        torch.cuda.synchronize()
        _barrier(world)
        step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
        # graph replays do not go through the library's launch counter: count
        # the kernels each captured step holds (persistent RK4 kernel +
        # bookkeeping, counted at capture)
        launches = int(lib.cdk_launch_count()) - l0 + per_step_launches * K
        eng.check()
        total_ms = _max_over_ranks(float(np.sum(step_ms)), world)

        # --- e2e: the public API with host arrays (a fresh model object: omega
        #     and theta0 uploaded from the host, the final state read back),
        #     inside the timed region; the decomposition's device graph is
        #     already resident (it is part of the problem setup, like the CSR)
        from paper_2203_16657_b200 import IntegrationPlan, integrate, kuramoto_model

        dec._cache["device_graph"] = dg
        e2e_times = []
        for rep in range(3):  # the first call builds the engine; min over the warm ones
            model = kuramoto_model(omega.copy(), case.coupling, case.n)
            flush_l2()
            torch.cuda.synchronize()
            t = time.perf_counter()
            tr = integrate(model, dec, theta0, IntegrationPlan(t_end=K * dt, dt=dt))
            final = tr.final
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t)
        e2e_s = min(e2e_times)
    clocks = sampler.summary()

    if not np.all(np.isfinite(final)):
        raise RuntimeError("non-finite final state")

    value = n * K / (total_ms / 1e3)
    b_rhs = algorithmic_bytes_per_rhs(n, nnz)
    ell = bool(dg.struct.ell_off)
    kernel = "ell_rk4_kernel" if ell else "kuramoto_rk4_kernel"
    # one launch of the timed kernel = one RK4 step = 4 RHS stages; its
    # duration is the timed step (the bookkeeping kernel adds ~2 us)
    launch_ms = float(np.mean(step_ms))
    peak, peak_kind = _peaks()
    achieved = 4 * b_rhs / (launch_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic_bytes(kernel)
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg2_config(case, dec),
        "setup": {"csr_device_bytes": dg.device_bytes(), "graph_gen_s": round(t_gen, 2),
                  "plan_build_s": round(t_plan, 2), "parallelism": "1 GPU"},
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_kind": peak_kind, "kernel": kernel,
            "algorithmic_bytes_per_launch": 4 * b_rhs,
            "algorithmic_bytes_per_rhs": b_rhs,
            "launch_ms_mean": launch_ms,
            "note": "one launch = one RK4 step (4 fused stages); achieved = 4 B_rhs / mean "
                    "timed step (CUDA events, L2 flushed before each step)",
        },
        "e2e": {"value": n * K / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(2 * 8 * n / K),
                "d2h_bytes_per_step": int(2 * 8 * n / K),
                "note": "integrate() via the public API: omega + theta0 from host, "
                        "initial + final states back to host; device graph already resident"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if ell and dg.schedule.ell is not None:
        res["l1_pipe"] = l1_pipe_floor(dg, n, launch_ms, clocks)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_sample(case, dec, omega, theta0, steps=args.cpu_steps)
    if rank == 0:
        print(json.dumps(res), flush=True)
    return 0


FP64_PEAK_TFLOPS = 36.4  # DFMA, measured on this pool (tools/fp64_peak.cu, profiles/r02_fp64_peak.txt)
CFG4_FLOP_PER_STEP = 2.5e9  # ncu SASS counts of the four stages (profiles/r02_experiments.txt)


def run_cfg34(args):
    """Secondary bench lines: config 3 (higher-order Kuramoto, triangles) and
    config 4 (Cucker-Smale, degree-8 P2).  Same contract as the config-2 line:
    W warm-up steps, K RK4 steps timed one by one with CUDA events and the L2
    flushed before each, e2e through the public integrate() with host arrays.
    Canonical bytes per RHS: cfg3 = 4 nnz_dir + 8 triangle incidences + 8 (N+1)
    + 24 N; cfg4 = 4 nnz_dir + 8 (N+1) + 64 N (state in, derivative out)."""
    import torch

    from paper_2203_16657_b200 import IntegrationPlan, _lib, configs, cs, ho, integrate

    torch.cuda.set_device(0)
    lib = _lib.lib()
    K = args.steps if args.steps != 2000 else 200
    W = max(3, args.warmup)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush_l2():
        flush.fill_(float(np.random.random()))

    t0 = time.perf_counter()
    if args.config == "cfg3":
        c = configs.config3()
        dec = c.decomposition()
        omega, x0 = c.state()
        eng = ho.HOEngine(dec, omega, c.k1, c.k2, norm=c.n)
        eng.set_state(x0)
        model = ho.ho_kuramoto_model(omega, c.k1, c.k2, norm=c.n)
        b_rhs = 4 * dec.nnz_dir + 8 * int(eng.graph.tri_pairs) + 8 * (c.n + 1) + 24 * c.n
        workload = ("cfg3 higher-order Kuramoto CIA RK4, SBM N=50000, 100 communities of 500, "
                    "p_in .9, p_out 1e-4, K1=1, K2=.5, dt .005")
        h2d = 2 * 8 * c.n
    else:
        c = configs.config4()
        dec = c.decomposition()
        pos, vel = c.state()
        model = cs.CuckerSmale(c.K, c.sigma, c.beta)
        eng = cs.CSEngine(dec, model, pos, vel, t_end=c.t_end)
        x0 = np.concatenate([pos, vel], axis=1)
        b_rhs = 4 * dec.nnz_dir + 8 * (c.n + 1) + 64 * c.n
        workload = ("cfg4 Cucker-Smale CIA RK4 (degree-8 P2 in squared distance), SBM N=100000, "
                    "100 communities of 1000, p_in .9, p_out 1e-4, dt .01")
        h2d = 4 * 8 * c.n
    t_setup = time.perf_counter() - t0
    sampler = ClockSampler(0)
    with sampler:
        eng.rk4(c.dt, W)
        torch.cuda.synchronize()
        l0 = int(lib.cdk_launch_count())
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        for k in range(K):
            flush_l2()
            starts[k].record()
            eng.rk4(c.dt, 1)
            ends[k].record()
        torch.cuda.synchronize()
        launches = int(lib.cdk_launch_count()) - l0
        eng.check()
        step_ms = np.array([a.elapsed_time(b) for a, b in zip(starts, ends)])
        e2e_times = []
        for rep in range(3):  # the first call builds the engine; min over the warm ones
            flush_l2()
            torch.cuda.synchronize()
            t = time.perf_counter()
            tr = integrate(model, dec, x0, IntegrationPlan(t_end=K * c.dt, dt=c.dt))
            final = tr.final
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t)
    clocks = sampler.summary()
    if not np.all(np.isfinite(final)):
        raise RuntimeError("non-finite final state")
    ms = float(step_ms.mean())
    peak, peak_kind = _peaks()
    achieved = 4 * b_rhs / (ms / 1e3) / 1e9
    res = {
        "metric": METRIC, "value": c.n / (ms / 1e3), "unit": UNIT, "n_gpus": 1, "steps": K,
        "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload, "n_nodes": c.n, "nnz_dir": int(dec.nnz_dir), "dt": c.dt,
                   "l2": "L2 flushed (512 MB write) before every timed step"},
        "setup": {"setup_s": round(t_setup, 2), "parallelism": "1 GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                     "kernel": "one RK4 step (4 stages of %s kernels)" %
                               ("ho_*" if args.config == "cfg3" else "cs_*"),
                     "algorithmic_bytes_per_rhs": int(b_rhs), "launch_ms_mean": ms,
                     "note": "achieved = 4 B_rhs / mean timed step; per-kernel ncu metrics in "
                             "profiles/r02_cfg34_final_ncu_launch_metrics.txt"},
        "e2e": {"value": c.n * K / min(e2e_times), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d / K), "d2h_bytes_per_step": int(h2d / K),
                "note": "integrate() via the public API with host arrays"},
        "gpu_launches": launches, "clocks": clocks, "cpu_baseline": None,
    }
    if args.config == "cfg4":
        tf = CFG4_FLOP_PER_STEP / (ms / 1e3) / 1e12
        res["fp64"] = {"achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                       "frac": tf / FP64_PEAK_TFLOPS,
                       "note": "flop per step from ncu SASS counts; peak = measured DFMA rate"}
    print(json.dumps(res), flush=True)
    return 0


def l1_pipe_floor(dg, n, launch_ms, clocks):
    """The bound that binds the ELL kernel: the SM's L1/shared
    data pipe moves one 128-byte wavefront per cycle, and every gather costs
    wavefronts whatever its bytes.  Counted from the layout, per RHS:
    window gathers 4 per LDS.128 of 32 slots; the chunk stream 8 per 32-lane
    chunk (4 written by cp.async into the ring, 4 read back); inter z gathers
    1 each (one 32-byte sector per lane) + their column loads; ~18 per rblock
    of epilogue loads/stores.  floor = wavefronts / (SMs x SM clock)."""
    import torch

    e, lay = dg.schedule.ell, dg.layout
    slots = int(e.slots())
    xslots = int(e.xell_col.shape[0])
    w_rhs = slots / 8 + slots / 32 + int(lay.nnz_inter) + xslots / 32 + 18 * lay.n_rblk
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = float(clocks.get("sm_mhz") or clocks.get("sm_max_mhz") or 0.0)
    floor_ms = 4 * w_rhs / (sms * mhz * 1e6) * 1e3 if mhz else None
    return {"unit": "128-byte wavefronts", "per_launch": int(4 * w_rhs),
            "gather_slots_per_rhs": slots, "sm_count": sms, "sm_mhz": mhz,
            "floor_ms": floor_ms, "frac": (floor_ms / launch_ms) if floor_ms else None,
            "note": "the HBM roofline does not bind this kernel (CSR stays in L2 across "
                    "stages); the L1/shared wavefront rate does: frac = floor / timed step"}


def cpu_baseline_cfg5(case, csr, dg, omega, theta0, rows: int = 20000):
    """Oracle C port on a bounded sample of config 5: one RHS with the full
    O(N) community terms and the directed corrections of the first ``rows``
    rows (as unordered pairs), extrapolated linearly in the pair count
    (CIA is O(N + nnz))."""
    from oracle import cia
    from oracle import kernels as K

    K.set_threads(1)
    off = case.offsets()
    iptr, xptr = csr.intra_ptr, csr.inter_ptr
    # device CSR: intra columns rebased to the segment windows (undo with the
    # schedule's per-row delta) and bank-ordered within runs
    icol = dg._t["intra_col"][: int(iptr[rows])].cpu().numpy().view(np.uint16)
    xcol = dg._t["inter_col"][: int(xptr[rows])].cpu().numpy().astype(np.int64)
    delta = dg.schedule.row_delta[:rows].astype(np.int64)
    ri = np.repeat(np.arange(rows), np.diff(iptr[: rows + 1]))
    keep = icol != 0xFFFF
    comm = np.searchsorted(off, np.arange(rows), side="right") - 1
    iu = np.concatenate([ri[keep], np.repeat(np.arange(rows), np.diff(xptr[: rows + 1]))])
    iv = np.concatenate([icol[keep].astype(np.int64) - delta[ri[keep]] + off[comm[ri[keep]]],
                         xcol])
    assert iv.min() >= 0 and iv.max() < case.n
    sg = np.concatenate([-np.ones(int(keep.sum())), np.ones(xcol.shape[0])])
    z = np.zeros(0, np.int64)

    def rhs(a, b, c):
        t = time.perf_counter()
        cia.kuramoto_rhs_cia(K, theta0, omega, off, a, b, c, case.coupling, case.n)
        return time.perf_counter() - t

    rhs(z, z, np.zeros(0))
    t0 = min(rhs(z, z, np.zeros(0)) for _ in range(2))
    t1 = rhs(iu, iv, sg)
    pairs_total = (csr.nnz_intra + int(xptr[-1])) / 2.0
    t_rhs = t0 + (t1 - t0) * pairs_total / iu.shape[0]
    return case.n / (4.0 * t_rhs), t1, iu.shape[0], t_rhs


def run_cfg5(args):
    """BASELINE configs[4] (LFR-style N = 8e6) on one GPU: device-generated
    graph (csrc/gen.cu), fused stage kernels, inputs (27 GB of CSR) far above
    L2, so no flush is needed between steps."""
    import torch

    rank, world, local = _dist_env()
    if world > 1 or os.environ.get("CDK_BENCH_SHARDED") == "1":
        from paper_2203_16657_b200 import multi

        return multi.bench_main(args)
    torch.cuda.set_device(local)
    from paper_2203_16657_b200 import _lib, gen
    from paper_2203_16657_b200.engine import KuramotoEngine

    lib = _lib.lib()
    case = gen.config5()
    omega, theta0 = case.state()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dg, csr = gen.device_graph(case, "cuda")
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    n = case.n
    nnz = csr.nnz_intra + int(csr.inter_ptr[-1])
    eng = KuramotoEngine(None, omega, coupling=case.coupling, norm=n, graph=dg)
    eng.set_state(theta0)
    dt = case.dt
    stream = torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    W, K = max(3, args.warmup), args.steps
    sampler = ClockSampler(local)
    with sampler:
        with torch.cuda.stream(stream):
            eng.rk4(dt, W, stream=stream)
        torch.cuda.synchronize()
        eng.set_state(theta0)
        torch.cuda.synchronize()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = int(lib.cdk_launch_count())
        start.record(cur)
        eng.rk4(dt, K)
        end.record(cur)
        torch.cuda.synchronize()
        launches = int(lib.cdk_launch_count()) - l0
        total_ms = start.elapsed_time(end)
        eng.check()
        # roofline pass: per-stage events
        eng.set_state(theta0)
        torch.cuda.synchronize()
        Kr = min(K, 10)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(Kr)]
        for i in range(Kr):
            ev[i][0].record(cur)
            for st_i in range(1, 5):
                eng.rk4_stage(dt, st_i)
                ev[i][st_i].record(cur)
        torch.cuda.synchronize()
        stage_ms = np.array([[ev[i][s_ - 1].elapsed_time(ev[i][s_]) for s_ in range(1, 5)]
                             for i in range(Kr)])
        # e2e: omega + theta0 from pinned host memory, K steps, final state back
        om_h = torch.from_numpy(omega).pin_memory()
        th_h = torch.from_numpy(theta0).pin_memory()
        out_h = torch.empty(n, dtype=torch.float64).pin_memory()
        torch.cuda.synchronize()
        t = time.perf_counter()
        eng.omega.copy_(om_h, non_blocking=True)
        eng.set_state(th_h.to("cuda", non_blocking=True))
        eng.rk4(dt, K)
        out_h.copy_(eng.theta, non_blocking=True)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t
    clocks = sampler.summary()
    value = n * K / (total_ms / 1e3)
    b_rhs = algorithmic_bytes_per_rhs(n, nnz)
    stage_mean_ms = float(stage_ms.mean())
    peak, peak_kind = _peaks()
    achieved = b_rhs / (stage_mean_ms / 1e3) / 1e9
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": K, "warmup": W,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (device-generated LFR-style)",
        "config": {
            "workload": "cfg5 Kuramoto CIA RK4, LFR-style N=8000000, power-law sizes [1e3,2e4], "
                        "p_in .9, mu .05, degree exponent 2.5, dt .01",
            "n_nodes": n, "n_comm": int(csr.n_comm), "nnz_dir": nnz,
            "csr_device_bytes": dg.device_bytes(), "l2": "inputs (CSR ~27 GB) >> L2; no flush",
            "graph_gen_plus_plan_s": round(t_gen, 2), "parallelism": "1 GPU",
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
            "kernel": "kuramoto_stage_kernel", "algorithmic_bytes_per_launch": b_rhs,
            "stage_ms_mean": stage_mean_ms,
            "stage_ms_by_stage": [float(x) for x in stage_ms.mean(axis=0)],
        },
        "e2e": {"value": n * K / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(16 * n / K),
                "d2h_bytes_per_step": int(8 * n / K),
                "note": "omega + theta0 from pinned host, K steps, final state to host"},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        rate, el, pairs, t_rhs = cpu_baseline_cfg5(case, csr, dg, omega, theta0)
        res["cpu_baseline"] = {
            "value": rate, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"one RHS with the corrections of the first 20000 rows ({pairs} pairs, "
                      f"{el:.1f} s), extrapolated linearly to all {nnz / 2:.3g} pairs "
                      f"({t_rhs:.0f} s per RHS); oracle C port, 1 thread"}
    print(json.dumps(res), flush=True)
    return 0


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` run directly: launch N ranks on this node exactly as
    the driver does (torch.distributed.run, 127.0.0.1, a free port); rank 0
    prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="cfg2", choices=["cfg2", "cfg3", "cfg4", "cfg5"],
                    help="cfg2 = the metric's config (default); cfg5 = the LFR-style N=8e6 "
                         "config (steps default 200); cfg3 / cfg4 = higher-order Kuramoto / "
                         "Cucker-Smale (secondary lines, steps default 200)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.config in ("cfg3", "cfg4"):
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "the reference ships no CIA "
                              "arithmetic for this model (its oracle here is a restatement of "
                              "the SPEC: tests/test_ho_oracle.py, tests/test_cs_oracle.py)"}))
            return 0
        return run_cfg34(args)
    if args.config == "cfg5":
        if args.impl != "reference" and (int(os.environ.get("WORLD_SIZE", "1")) > 1
                                         or os.environ.get("CDK_BENCH_SHARDED") == "1"):
            return run_ours(args)
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "cfg5 reference arm not run: "
                              "~4 CPU-minutes per RHS; see cpu_baseline of the cfg5 line"}))
            return 0
        return run_cfg5(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
