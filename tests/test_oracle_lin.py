"""Pins of the single-loop linearised ADMM scheme of the oracle (SURVEY §8(f) NEXT-2,
oracle/msa_oracle.c mo_iteration_lin): each check is fixed by the mathematics, not by the
oracle itself.
  L1  dt = 0: the fixed point is the ROF minimiser of an independent Chambolle dual-projection
      solver (1e-9) and no random perturbation lowers K (eq:cost_TV).
  L2  one step equals the Alg. 2 v- and mu-updates with gamma = rho (eq:soft_threshold, line 7)
      followed by a linearised prox step on eq:new_adjoint's gradient, written out here from the
      paper's formulas with numpy (an independent transcription, not a re-call of the oracle).
  L3  constant image: c = I, mu = 0 bitwise for every iteration.
  L4  per-channel mean preserved (sum div = 0, antisymmetric agent term), with the agent on.
  L5  weak duality of the round record: mu stays in the beta-ball, so p = -mu is ROF-dual
      feasible and gap = K - D >= 0 at every round; gap -> 0 with dt = 0.
  L6  step-size rule: default tau = 0.99/(rho L^2); tau rho L^2 >= 1 and kappa > 1 are rejected."""
import numpy as np
import pytest

import oracle

from test_oracle_pins import _chambolle_rof, _np_div, _np_grad  # noqa: F401  (independent numpy stencils)


def _params(H, W, C, **kw):
    h = 1.0 / (W - 1)
    base = dict(height=H, width=W, channels=C, radius=2, eps_c=57.0, dt=0.25, alpha=8.0 / h, beta=1.0,
                rho=2.5 * h, gamma=2.5 * h, iters_per_round=10, rounds=3, scheme=1)
    base.update(kw)
    return oracle.Params(**base)


def test_L1_dt0_reaches_rof_minimiser():
    rng = np.random.default_rng(171)
    H = W = 8
    C = 3
    I = rng.random((H, W, C))
    h = 1.0 / 7
    prm = _params(H, W, C, dt=0.0, rho=2.5 * h * 40, gamma=2.5 * h * 40, iters_per_round=1000, rounds=100)
    s = oracle.solve(prm, I)
    d = oracle.derive(prm)
    ref = _chambolle_rof(I, prm.alpha, prm.beta, d.hx, d.hy, iters=400000)
    assert np.max(np.abs(s.c - ref)) <= 1e-12
    K0 = oracle.energy_K(prm, s.c, I)
    for _ in range(1000):
        dvec = rng.standard_normal(I.shape)
        dvec /= np.linalg.norm(dvec)
        for step in (1e-2, -1e-2, 1e-3, -1e-3):
            assert oracle.energy_K(prm, s.c + step * dvec, I) >= K0 - 1e-12
    assert abs(s.stats[-1][4]) <= 1e-12  # duality gap closed


def _shrink(a, t):
    n = np.linalg.norm(a, axis=-1, keepdims=True)
    return np.maximum(0.0, 1.0 - t / np.maximum(n, 1e-300)) * a


def test_L2_one_step_is_alg2_with_gamma_rho_and_a_linearised_prox():
    rng = np.random.default_rng(172)
    H, W, C = 7, 9, 3
    I = rng.random((H, W, C))
    prm = _params(H, W, C)
    d = oracle.derive(prm)
    s = oracle.State(prm, I)
    s.c = I + 0.05 * rng.standard_normal(I.shape)
    s.mu = 0.3 * rng.standard_normal((H, W, 2 * C))
    c0, mu0 = s.c.copy(), s.mu.copy()
    rho, tau, alpha = prm.rho, d.tau, prm.alpha
    # reference, from the paper's formulas
    F = oracle.agent_rhs(prm, c0)
    chalf = c0 + prm.dt * F
    g = _np_grad(c0, d.hx, d.hy)
    v = _shrink(g - mu0 / rho, prm.beta / rho)            # eq:soft_threshold, a = grad u - mu/rho
    mu1 = mu0 + prm.gamma * (v - g)                        # Alg. 2 line 7, gamma = rho
    smooth_grad = _np_div(mu1 + rho * v - rho * g, d.hx, d.hy)  # eq:new_adjoint's div(mu + rho v - rho grad u), updated mu, v
    c1 = (chalf - tau * smooth_grad + tau * alpha * I) / (1.0 + tau * alpha)  # linearised prox step
    s.run(1)
    assert np.max(np.abs(s.mu - mu1)) <= 1e-12
    assert np.max(np.abs(s.c - c1)) <= 1e-12


def test_L3_constant_image_fixed_point_bitwise():
    I = np.tile(np.array([0.25, 0.5, 0.875]), (9, 11, 1))
    s = oracle.State(_params(9, 11, 3), I)
    for _ in range(4):
        s.run(5)
        assert np.array_equal(s.c, I)
        assert not np.any(s.mu)


def test_L4_mean_preserved():
    rng = np.random.default_rng(174)
    I = rng.random((14, 17, 3))
    s = oracle.State(_params(14, 17, 3, eps_c=5.0, radius=3), I)
    s.run(100)
    assert np.allclose(s.c.reshape(-1, 3).mean(0), I.reshape(-1, 3).mean(0), rtol=1e-12, atol=0)


def test_L5_weak_duality_and_gap_closing():
    rng = np.random.default_rng(175)
    H = W = 12
    I = rng.random((H, W, 3))
    s = oracle.State(_params(H, W, 3, iters_per_round=20, rounds=10), I)
    s.run(200)
    assert np.all(np.linalg.norm(s.mu, axis=-1) <= 1.0 + 1e-12)
    for st in s.stats:
        assert st[4] >= -1e-12
    s0 = oracle.State(_params(H, W, 3, dt=0.0, iters_per_round=5, rounds=400), I)
    s0.run(2000)
    gaps = [st[4] for st in s0.stats]
    assert min(gaps) >= -1e-12
    assert gaps[-1] <= 1e-6 * gaps[0] and gaps[-1] <= 1e-8


def test_L6_step_size_rule():
    prm = _params(6, 6, 3)
    d = oracle.derive(prm)
    L2 = 4 / d.hx ** 2 + 4 / d.hy ** 2
    assert d.tau == pytest.approx(0.99 / (prm.rho * L2), rel=1e-15)
    with pytest.raises(ValueError):
        oracle.derive(_params(6, 6, 3, tau=1.0 / (prm.rho * L2)))
    with pytest.raises(ValueError):
        oracle.derive(_params(6, 6, 3, kappa=1.5))
