"""Config 2: a few standalone RK4 stage-2 launches (ncu target; stage 2 reads
L2-warm state like stages 2-4 of a timed step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_16657_b200 import configs  # noqa: E402
from paper_2203_16657_b200.engine import KuramotoEngine  # noqa: E402

c = configs.config2()
dec = c.decomposition()
omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
eng.set_state(theta0)
for _ in range(int(os.environ.get("N_STAGE", "3"))):
    eng.rk4_stage(c.dt, 1)
    eng.rk4_stage(c.dt, 2)
torch.cuda.synchronize()
print("ok")
