"""Configs 3 (higher-order Kuramoto, triangles) and 4 (Cucker-Smale, degree-8
polynomial P2) on one GPU: device-resident RK4 steps timed with CUDA events
(warm-up first), node-updates/s.  Not bench lines (BASELINE's metric is quoted
on config 2); measurements for DESIGN.md.

    python tools/bench_cfg34.py [--steps 50] [--only cfg3|cfg4]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_16657_b200 import configs, cs, ho  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--only", default="")
args = ap.parse_args()


def timed(step, k):
    step(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step(k)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


res = {}
if args.only in ("", "cfg3"):
    c = configs.config3()
    t = time.perf_counter()
    dec = c.decomposition()
    omega, theta0 = c.state()
    eng = ho.HOEngine(dec, omega, c.k1, c.k2, norm=c.n)
    t_plan = time.perf_counter() - t
    eng.set_state(theta0)
    ms = timed(lambda k: eng.rk4(c.dt, k), args.steps)
    eng.check()
    res["cfg3"] = {"n": c.n, "ms_per_step": ms, "node_updates_per_s": c.n / (ms / 1e3),
                   "setup_s": round(t_plan, 2)}
if args.only in ("", "cfg4"):
    c = configs.config4()
    t = time.perf_counter()
    dec = c.decomposition()
    pos, vel = c.state()
    model = cs.CuckerSmale(c.K, c.sigma, c.beta)
    eng = cs.CSEngine(dec, model, pos, vel, t_end=c.t_end)
    t_plan = time.perf_counter() - t
    ms = timed(lambda k: eng.rk4(c.dt, k), args.steps)
    eng.check()
    res["cfg4"] = {"n": c.n, "ms_per_step": ms, "node_updates_per_s": c.n / (ms / 1e3),
                   "setup_s": round(t_plan, 2)}
print(json.dumps(res))
