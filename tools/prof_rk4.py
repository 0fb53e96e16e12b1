"""Stage timeline of the persistent ELL RK4 kernel (CDK_PROFILE build): per
CTA, globaltimer at the start and end of each stage of the second step ->
stage work (max over CTAs) vs grid-barrier release gaps."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
os.environ.setdefault("CDK_LIB", os.path.join(REPO, "paper_2203_16657_b200/_build/libcommdyn_cuda_profile.so"))
import numpy as np, torch
from paper_2203_16657_b200 import configs
from paper_2203_16657_b200.engine import KuramotoEngine
c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
n_cta = eng.graph.schedule.n_cta
prof = torch.zeros(18 * n_cta, dtype=torch.int64, device="cuda")
eng.lib.cdk_debug_set_profile_buffer(prof.data_ptr())
eng.set_state(theta0)
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); eng.rk4(c.dt, 3); ev[1].record()
    torch.cuda.synchronize()
    print(f"rep {rep}: 3 RK4 steps {ev[0].elapsed_time(ev[1])*1e3:.1f} us")
T = prof[6 * n_cta:14 * n_cta].view(n_cta, 8).cpu().numpy().astype(np.float64)
D = prof[14 * n_cta:].view(n_cta, 4).cpu().numpy().astype(np.float64)
print(f"intra-CTA drain: {D[:, 0].sum() / max(D[:, 1].sum(), 1):.3f} of warp time after segment ready "
      f"({D[:, 2].sum():.0f} segments)")
T -= T.min()
for st in range(4):
    s0, s1 = T[:, 2 * st], T[:, 2 * st + 1]
    print(f"stage {st+1}: start min {s0.min()/1e3:.2f} max {s0.max()/1e3:.2f}  end min {s1.min()/1e3:.2f} "
          f"p50 {np.median(s1)/1e3:.2f} max {s1.max()/1e3:.2f} us; work mean {np.mean(s1-s0)/1e3:.2f} max {np.max(s1-s0)/1e3:.2f}")
