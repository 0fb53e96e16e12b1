"""Stability of per-CTA stage cycles across launches (CDK_PROFILE build):
correlation between two launches, and against the planner's cost model."""
import os, sys
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
os.environ.setdefault("CDK_LIB", os.path.join(REPO, "paper_2203_16657_b200/_build/libcommdyn_cuda_profile.so"))
import numpy as np, torch
from paper_2203_16657_b200 import configs, plan as PL
from paper_2203_16657_b200.engine import KuramotoEngine
c = configs.config2(); dec = c.decomposition(); omega, theta0 = c.state()
eng = KuramotoEngine(dec, omega, coupling=c.coupling, norm=c.n)
sch = eng.graph.schedule; lay = eng.graph.layout; e = sch.ell
prof = torch.zeros(6 * sch.n_cta, dtype=torch.int64, device="cuda")
eng.lib.cdk_debug_set_profile_buffer(prof.data_ptr())
eng.set_state(theta0)
runs = []
for it in range(4):
    eng.rk4_stage(c.dt, 1 + (it % 4))
    torch.cuda.synchronize()
    runs.append(prof.view(-1, 6)[:, 0].cpu().numpy().astype(np.float64))
R = np.array(runs)
print("per-launch mean/max:", [(int(r.mean()), int(r.max())) for r in R])
for a in range(4):
    print("corr with launch 0:", round(float(np.corrcoef(R[0], R[a])[0, 1]), 3))
seg_rb = sch.seg_rblk
e_off, e_nch, x_off = PL._ell_sizes(lay)[0], None, PL._ell_sizes(lay)[1]
cost = []
for b in range(sch.n_cta):
    a_, z = seg_rb[sch.cta_seg[b]], seg_rb[sch.cta_seg[b + 1]]
    cost.append(8 * (e.ell_off[z] - e.ell_off[a_]) * PL.ELL_SLOT_COST + (e.xell_off[z] - e.xell_off[a_]) * PL.ELL_XSLOT_COST + (z - a_) * PL.ELL_RBLK_COST)
cost = np.array(cost)
print("corr model vs measured:", round(float(np.corrcoef(cost, R.mean(0))[0, 1]), 3), "model spread", cost.min(), cost.max())
