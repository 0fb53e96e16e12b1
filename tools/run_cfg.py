"""Small driver for profiling: build a config, run a few fused RK4 steps.

    python tools/run_cfg.py [--config cfg2] [--steps 3] [--rhs]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2203_16657_b200 import configs  # noqa: E402
from paper_2203_16657_b200.engine import KuramotoEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
c = configs.CONFIGS[a.config]()
dec = c.decomposition()
omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
eng.set_state(theta0)
eng.rk4(c.dt, a.steps)
torch.cuda.synchronize()
eng.check()
print("ok", eng.theta[:4].tolist())
