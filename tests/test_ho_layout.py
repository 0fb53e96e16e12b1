"""Host layout of the higher-order kernels (CPU): the CTA work table covers
every rblock once, one community (or the pool) per CTA, with that
community's node window."""

import numpy as np

from paper_2203_16657_b200 import configs, ho, plan


def test_cta_table():
    c = configs.scaled_config3(m=6, lam=100, p_out=3e-3)
    dec = c.decomposition()
    lay = plan.build_layout(dec)
    cta_rb, cta_win, win_cap = ho.ho_cta_table(lay)
    assert cta_rb[0] == 0 and cta_rb[-1] == lay.n_rblk and np.all(np.diff(cta_rb) >= 1)
    assert np.all(np.diff(cta_rb) <= ho.HO_CTA_RBLK)
    off = lay.comm_off
    for q in range(cta_rb.shape[0] - 1):
        comms = set(lay.rblk_comm[cta_rb[q]: cta_rb[q + 1]].tolist())
        assert len(comms) == 1
        cc = comms.pop()
        if cc >= 0:
            assert tuple(cta_win[q]) == (off[cc], off[cc + 1])
    assert win_cap == int(np.diff(off).max())
