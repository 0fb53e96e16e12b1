import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200.engine import KuramotoEngine
c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
k = eng.rhs(torch.from_numpy(theta0).cuda()); torch.cuda.synchronize(); print("rhs ok", float(k.sum()))
eng.set_state(theta0); eng.rk4(c.dt, 2); torch.cuda.synchronize(); print("rk4 ok")
