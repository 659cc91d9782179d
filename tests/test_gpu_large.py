"""Large interaction supports (msa_agent_large.cu): the paper's control box
E = [2, 1100]^2 gives supports of many pixels, where step 1 is an n-body-style sum.
  * the chunked shared-memory kernel against the generic kernel (same weights, other summation
    order): p+ of one iteration bitwise, c to fp32 rounding; three iterations across a round;
  * parity with the oracle for a windowed run with the default eps_x (support = R) and for a small
    eps_x inside E whose support fits the window, so the window sum is the paper's all-pairs sum
    (pin P7); both iteration schemes."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from _harness import rel_err_per_pixel, hook_env

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(spec, variant, tmp_path):
    out = str(tmp_path / f"{variant}.npz")
    env = hook_env(MSA_K1=variant)
    env.pop("MSA_FORCE_GENERIC", None)
    subprocess.run([sys.executable, os.path.join(HERE, "_run_case.py"), json.dumps(spec), out], check=True, env=env)
    return np.load(out)


@pytest.mark.parametrize("shape,R,ker,scheme", [((1, 48, 40, 3), 6, 0, 0), ((1, 41, 37, 1), 8, 1, 0),
                                                ((1, 48, 40, 3), 9, 0, 0), ((1, 70, 66, 3), 16, 0, 0),
                                                ((2, 37, 29, 3), 12, 1, 0), ((1, 90, 50, 1), 24, 0, 0),
                                                ((1, 64, 64, 3), 40, 0, 0), ((1, 66, 70, 3), 16, 0, 1),
                                                ((1, 40, 41, 4), 20, 0, 0)])
def test_large_kernel_matches_generic(shape, R, ker, scheme, tmp_path):
    B, H, W, C = shape
    h = 1.0 / (W - 1)
    base = dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=ker, eps_c=20.0, dt=0.25, rho=2.5 * h, gamma=2.5 * h,
                iters_per_round=2, rounds=1, scheme=scheme)
    for iters, tol in ((1, 2e-6), (3, 2e-5)):
        spec = dict(seed=H * 7 + W + R, shape=list(shape), iters=iters, params=base)
        a = _run(spec, "generic", tmp_path)
        b = _run(spec, "tile", tmp_path)
        if iters == 1 and scheme == 0:
            assert np.array_equal(a["p"], b["p"])
        for k in ("c", "p") if scheme == 0 else ("c", "mu"):
            scale = max(1.0, float(np.max(np.abs(a[k]))))
            assert np.max(np.abs(a[k] - b[k])) / scale <= tol, (iters, k)


@pytest.mark.parametrize("eps_x,R,scheme", [(0.0, 16, 0), (50.0, 16, 0), (50.0, 16, 1), (0.0, 10, 1)])
def test_large_support_parity_with_oracle(eps_x, R, scheme):
    rng = np.random.default_rng(int(eps_x) + R + 10 * scheme)
    H, W, C = 64, 64, 3
    I = np.clip(rng.random((1, H, W, C)) * 0.2 + np.repeat(np.repeat(rng.random((1, 4, 4, C)), 16, 1), 16, 2), 0, 1)
    I = I.astype(np.float32)
    h = 1.0 / (W - 1)
    sp = dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=0, eps_x=eps_x, eps_c=57.0, dt=0.25, rho=2.5 * h,
              gamma=2.5 * h, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=25, rounds=2, scheme=scheme)
    if eps_x > 0:  # the support radius in pixels must fit the window: then window sum = all-pairs sum (P7)
        assert 1.0 / (h * np.sqrt(eps_x / 2.0)) < R
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I) as s:
        s.solve()
        gc = s.get_field(msa.FIELD_C)[0]
    o = oracle.State(oracle.Params.from_solver(H, W, C, sp), I[0].astype(np.float64))
    o.run(50)
    assert np.max(rel_err_per_pixel(gc, o.c)) <= 1e-4


@pytest.mark.parametrize("H,W,C,R,eps_x", [(48, 48, 1, 100, 2.0), (36, 30, 3, 255, 2.0), (80, 72, 2, 140, 2.0)])
def test_all_pairs_regime_parity_with_oracle(H, W, C, R, eps_x):
    """The paper's box E = [2, 1100]^2 at its lower end (eps_x = 2): supports of the whole image.
    With R >= the support radius (up to the new R <= 255) the window sum is the paper's all-pairs
    sum with 1/N_R, which the oracle evaluates pair by pair."""
    rng = np.random.default_rng(H + W + C + R)
    I = np.clip(rng.random((1, H, W, C)) * 0.2 + np.repeat(np.repeat(rng.random((1, 3, 3, C)), H // 3 + 1, 1)[:, :H],
                                                          W // 3 + 1, 2)[:, :, :W], 0, 1).astype(np.float32)
    h = 1.0 / (max(W, H) - 1)
    assert 1.0 / (h * np.sqrt(eps_x / 2.0)) <= R or R >= max(H, W)
    sp = dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=0, eps_x=eps_x, eps_c=57.0, dt=0.25, rho=2.5 * h,
              gamma=2.5 * h, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=5, rounds=2, scheme=0)
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I) as s:
        s.solve()
        gc = s.get_field(msa.FIELD_C)[0]
    o = oracle.State(oracle.Params.from_solver(H, W, C, sp), I[0].astype(np.float64))
    o.run(10)
    assert np.max(rel_err_per_pixel(gc, o.c)) <= 1e-4
