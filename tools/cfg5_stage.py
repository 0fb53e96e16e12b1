"""Generate config 5 on the device and run a few stage-1 launches (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_16657_b200 import gen  # noqa: E402
from paper_2203_16657_b200.engine import KuramotoEngine  # noqa: E402

small = "--small" in sys.argv
c = gen.config5() if not small else gen.scaled_config5(400_000, 1000, 20000)
omega, theta0 = c.state()
dg, _ = gen.device_graph(c, "cuda")
eng = KuramotoEngine(None, omega, coupling=c.coupling, norm=c.n, graph=dg)
eng.set_state(theta0)
for _ in range(int(os.environ.get("N_STAGE", "3"))):
    eng.rk4_stage(c.dt, 1)
torch.cuda.synchronize()
print("ok", c.n, dg.schedule.n_seg)
