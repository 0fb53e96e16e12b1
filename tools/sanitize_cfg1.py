"""compute-sanitizer target: config 1 through the persistent RK4 kernels
(ELL: ell_rk4_kernel; CDK_ELL=0: kuramoto_rk4_kernel), plus one RHS and the
per-stage launches, 3 steps each; parity vs the golden trajectory prefix is
checked by the GPU tests, here only that the run completes and is finite."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2203_16657_b200 import configs  # noqa: E402
from paper_2203_16657_b200.engine import KuramotoEngine  # noqa: E402

c = configs.config1()
dec = c.decomposition()
omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
print("kernel family:", "ell" if eng.graph.struct.ell_off else "row-group")
k = eng.rhs(torch.from_numpy(theta0).cuda())
eng.set_state(theta0)
eng.rk4(c.dt, 3)
for st in range(1, 5):
    eng.rk4_stage(c.dt, st)
eng.check()
torch.cuda.synchronize()
assert np.all(np.isfinite(eng.theta.cpu().numpy())) and bool(torch.isfinite(k).all())
print("ok")
