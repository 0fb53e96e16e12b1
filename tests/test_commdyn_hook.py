"""The drop-in proved through the reference itself: the INTEGRATION.md §2
binding (paper_2203_16657_b200/commdyn_hook.py) installed on the UNMODIFIED
reference package — baseline/_ref/commdyn (pip --target install, git-ignored,
shipped to the GPU box) or, in the build container, /root/reference — and the
reference's OWN dispatchers run with COMMDYN_BACKEND=cuda.

Each case runs in a fresh interpreter (the binding mutates the imported
reference modules).  CPU tests: the switch (cuda <-> numba <-> numpy, the
reference's ValueError kept), the wrapped dispatchers, and that a cuda call
without a GPU fails loudly (no silent CPU fallback).  GPU tests: every
wrapped dispatcher vs the golden fixtures, the SPEC orchestration over the
reference's dispatchers for config 1 (1000 RK4 steps) vs the golden
trajectory, and flipping back to numba mid-process.
"""

import os
import subprocess
import sys
import textwrap

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_path():
    for p in (os.path.join(REPO, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isfile(os.path.join(p, "commdyn", "_kernels.py")):
            return p
    return None


def _run(code: str, env_extra: dict | None = None, timeout: int = 600):
    ref = _ref_path()
    if ref is None:
        pytest.skip("reference package not installed (baseline/_ref) and /root/reference absent")
    env = dict(os.environ)
    env.pop("COMMDYN_BACKEND", None)
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/commdyn_numba_cache")
    env.update(env_extra or {})
    prelude = textwrap.dedent(f"""
        import sys
        sys.path.insert(0, {REPO!r})
        REF = {ref!r}
        GOLDEN = {os.path.join(REPO, "tests", "golden")!r}
    """)
    res = subprocess.run([sys.executable, "-c", prelude + textwrap.dedent(code)], env=env,
                         capture_output=True, text=True, timeout=timeout)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-3000:]
    return res.stdout


def test_switch_and_wrapped_dispatchers():
    out = _run("""
        import numpy as np
        from paper_2203_16657_b200 import commdyn_hook as H
        rb, rk = H.import_commdyn(REF)
        assert rb.__file__.startswith(REF), rb.__file__
        assert rb.backend() == "numba"
        for name in H.DISPATCHERS:
            fn = getattr(rk, name)
            assert fn.__name__ == name and hasattr(fn, "__wrapped_reference__"), name
        assert not hasattr(rk.pairs_callable, "__wrapped_reference__")
        rb.set_backend("numpy"); assert rb.backend() == "numpy" and not rb.USE_NUMBA
        rb.set_backend("numba"); assert rb.backend() == "numba" and rb.USE_NUMBA
        try:
            rb.set_backend("fortran")
        except ValueError:
            pass
        else:
            raise AssertionError("unknown backend accepted")
        import torch
        from paper_2203_16657_b200.errors import DeviceError
        if torch.cuda.is_available():
            rb.set_backend("cuda")
            assert rb.backend() == "cuda" and rb.USE_CUDA
        else:  # no GPU: the switch refuses loudly and the reference backend stays active
            try:
                rb.set_backend("cuda")
            except DeviceError:
                pass
            else:
                raise AssertionError("cuda backend selected without a GPU")
            assert rb.backend() == "numba" and not rb.USE_CUDA
        rb.set_backend("numba")
        assert rb.backend() == "numba" and not rb.USE_CUDA
        # a reference-backend call is untouched by the binding
        x = np.linspace(-3, 3, 10); off = np.array([0, 4, 10])
        r = rk.order_params_blocks(x, off, 1, np.pi, 10)
        assert r.shape == (2, 3)
        H.install(rb, rk)  # idempotent
        print("OK")
    """)
    assert "OK" in out


def test_env_cuda_selects_device_backend_or_fails_loudly():
    out = _run("""
        import os, torch
        from paper_2203_16657_b200 import commdyn_hook as H
        from paper_2203_16657_b200.errors import DeviceError
        if torch.cuda.is_available():
            rb, rk = H.import_commdyn(REF)
            assert rb.backend() == "cuda", rb.backend()
        else:
            try:
                H.import_commdyn(REF)
            except DeviceError as e:
                print("LOUD", e)
            else:
                raise AssertionError("COMMDYN_BACKEND=cuda accepted without a GPU")
        assert os.environ["COMMDYN_BACKEND"] == "cuda"
        print("OK")
    """, {"COMMDYN_BACKEND": "cuda"})
    assert "OK" in out


@pytest.mark.gpu
def test_reference_dispatchers_on_cuda_vs_golden():
    out = _run("""
        import math, os
        import numpy as np
        from paper_2203_16657_b200 import commdyn_hook as H
        rb, rk = H.import_commdyn(REF)
        assert rb.backend() == "cuda"
        ks = dict(np.load(os.path.join(GOLDEN, "kernels_small.npz")))
        f4 = dict(np.load(os.path.join(GOLDEN, "kernels_f4.npz")))
        x, off = ks["x"], ks["offsets"]; n = x.shape[0]
        TOL = 1e-12
        def close(a, b, tol=TOL):
            assert np.abs(np.asarray(a) - np.asarray(b)).max() <= tol, np.abs(a - b).max()
        for p in (1, 2, 3):
            close(rk.order_params_blocks(x, off, p, math.pi, n), ks[f"op_p{p}"])
        o = ks["dc_out0"].copy()
        nv, mi = rk.dense_complex(x, off, ks["dc_tbl"], math.pi, o)
        close(o, ks["dc_out"]); assert nv == 0
        o = np.zeros(n); rk.dense_real(x, off, ks["dr_tc"], ks["dr_ts"], math.pi, o)
        close(o, ks["dr_out"])
        o = np.zeros(n)
        rk.pairs_trig(ks["pt_iu"], ks["pt_iv"], x, 1.0 / n, ks["pt_dcos"], ks["pt_dsin"],
                      math.pi, ks["pt_sgn"], o)
        close(o, ks["pt_out"])
        o = np.zeros((n, 2))
        rk.pairs_cs(ks["pt_iu"], ks["pt_iv"], ks["cs_pos"], ks["cs_vel"], 1.0 / n, 1.0, 1.0,
                    0.25, ks["pt_sgn"], o)
        close(o, ks["cs_out"])
        close(rk.moments_blocks(x, off, 5, 0.3, n), ks["mom"])
        o = np.zeros(n); rk.dense_poly(x, off, ks["dp_tbl"], 0.5, -0.1, o)
        close(o, ks["dp_out"])
        close(rk.ho_naive_block(ks["ho_theta"], (1, 1, 0, -2)), ks["ho_1102"])
        o = f4["pp_out0"].copy(); m = o.shape[0]
        rk.pairs_poly(f4["pp_iu"], f4["pp_iv"], f4["pp_x"], 1.0 / m, f4["pp_coef"], 0.2,
                      f4["pp_sgn"], o)
        close(o, f4["pp_out"])
        ph = f4["nn_b_ph"]
        assert np.array_equal(rk.nn_recurrence(ph, int(f4["nn_b_k"]), 1.0 / ph.shape[0],
                                               int(f4["nn_b_anchor"])), f4["nn_b_f"])
        assert np.array_equal(rk.spin_field_sums(f4["spin"]), f4["spin_f"])
        # back to the reference's own numba kernels in the same process
        rb.set_backend("numba")
        assert rb.backend() == "numba"
        close(rk.order_params_blocks(x, off, 2, math.pi, n), ks["op_p2"], 1e-13)
        print("OK")
    """, {"COMMDYN_BACKEND": "cuda"})
    assert "OK" in out


@pytest.mark.gpu
def test_reference_orchestration_on_cuda_config1_1000_steps():
    """oracle/cia.py's SPEC orchestration composed ONLY of the reference's
    dispatchers (as a SPEC-level caller of commdyn would), backend cuda:
    config 1, 1000 RK4 steps vs the golden CIA and direct-sum trajectories."""
    out = _run("""
        import os
        import numpy as np
        from oracle import cia
        from paper_2203_16657_b200 import commdyn_hook as H, configs
        rb, rk = H.import_commdyn(REF)
        assert rb.backend() == "cuda"
        c = configs.config1()
        dec = c.decomposition()
        omega, theta0 = c.state()
        s = dec.correction
        g = np.load(os.path.join(GOLDEN, "cfg1.npz"))
        def rhs(x):
            return cia.kuramoto_rhs_cia(rk, x, omega, dec.offsets, s.iu, s.iv, s.sgn,
                                        c.coupling, c.n)
        k0 = rhs(theta0)
        assert np.abs(k0 - g["rhs0_cia"]).max() <= 1e-12
        fin, _ = cia.rk4_integrate(rhs, theta0, c.dt, c.steps)
        assert cia.circ_dist(fin, g["final_cia"]).max() <= 1e-9
        assert cia.circ_dist(fin, g["final_naive"]).max() <= 1e-9
        print("OK")
    """, {"COMMDYN_BACKEND": "cuda"}, timeout=900)
    assert "OK" in out
