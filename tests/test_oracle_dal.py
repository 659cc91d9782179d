"""Pins of the DAL oracle (Algorithm 1; oracle mo_dal*):
  D1  phi' against a central difference of phi (both kernel forms, eq:kernel).
  D2  the transpose Jacobian product (eq:dF_dc, R26) against the directional derivative of F by
      central differences: <g, v> = d/dh <lam, F(c + h v)>.
  D3  <lam, dF/deps> (eq:dF_depsx, eq:dF_depsc) against central differences in eps.
  D4  the full discrete-adjoint gradient of J against central differences of J, for the quadratic
      cost (eq:cost_functional) and the L~ cost with v, mu (eq:complete_square, eq:new_adjoint).
  D5  Algorithm 1: every accepted step satisfies the Armijo test, J never increases, eps stays in E."""
import numpy as np
import pytest

import oracle


def _setup(H=6, W=7, C=3, R=3, M=4, seed=0, **kw):
    rng = np.random.default_rng(seed)
    I = rng.random((H, W, C))
    p = oracle.Params(height=H, width=W, channels=C, radius=R, eps_x=30.0, eps_c=8.0, dt=0.25, alpha=5.0,
                      beta=1.0, rho=1.0, gamma=1.0, **kw)
    eps = np.stack([rng.uniform(20.0, 60.0, M), rng.uniform(4.0, 12.0, M)], axis=1)
    return rng, I, p, eps


@pytest.mark.parametrize("kernel", [0, 1])
def test_D1_phi_prime(kernel):
    for r in np.linspace(0.01, 0.99, 23):
        h = 1e-6
        fd = (oracle.phi(r + h, kernel) - oracle.phi(r - h, kernel)) / (2 * h)
        assert oracle.phi_prime(r, kernel) == pytest.approx(fd, rel=1e-7, abs=1e-9)
    assert oracle.phi_prime(1.0, kernel) == 0.0 and oracle.phi_prime(1.5, kernel) == 0.0


@pytest.mark.parametrize("C,kernel", [(3, 0), (1, 1), (2, 0)])
def test_D2_transpose_jacobian_product(C, kernel):
    rng, I, p, _ = _setup(C=C, kernel=kernel)
    c = I + 0.05 * rng.standard_normal(I.shape)
    lam = rng.standard_normal(I.shape)
    v = rng.standard_normal(I.shape)
    ex, ec = 30.0, 8.0
    g = oracle.agent_jtvp(p, ex, ec, c, lam)
    h = 1e-6
    fd = (np.sum(lam * oracle.agent_rhs_eps(p, ex, ec, c + h * v)) -
          np.sum(lam * oracle.agent_rhs_eps(p, ex, ec, c - h * v))) / (2 * h)
    assert np.sum(g * v) == pytest.approx(fd, rel=1e-7)


def test_D3_eps_derivatives():
    rng, I, p, _ = _setup()
    c = I + 0.05 * rng.standard_normal(I.shape)
    lam = rng.standard_normal(I.shape)
    ex, ec = 30.0, 8.0
    de = oracle.agent_deps(p, ex, ec, c, lam)
    h = 1e-5
    fx = (np.sum(lam * oracle.agent_rhs_eps(p, ex + h, ec, c)) - np.sum(lam * oracle.agent_rhs_eps(p, ex - h, ec, c)))
    fc = (np.sum(lam * oracle.agent_rhs_eps(p, ex, ec + h, c)) - np.sum(lam * oracle.agent_rhs_eps(p, ex, ec - h, c)))
    assert de[0] == pytest.approx(fx / (2 * h), rel=1e-6)
    assert de[1] == pytest.approx(fc / (2 * h), rel=1e-6)


@pytest.mark.parametrize("cost", [0, 1])
def test_D4_gradient_matches_finite_differences(cost):
    rng, I, p, eps = _setup(M=5, seed=3 + cost)
    d = oracle.DalParams(M=5, cost=cost, rho=0.7)
    v = mu = None
    if cost == 1:
        v = 0.3 * rng.standard_normal((6, 7, 6))
        mu = 0.3 * rng.standard_normal((6, 7, 6))
    J, g = oracle.dal_gradient(p, d, eps, I, v, mu)
    assert J == pytest.approx(oracle.dal_cost(p, d, eps, I, v, mu), rel=1e-15)
    for m in range(5):
        for q in range(2):
            h = 1e-4 * eps[m, q]
            ep, em = eps.copy(), eps.copy()
            ep[m, q] += h
            em[m, q] -= h
            fd = (oracle.dal_cost(p, d, ep, I, v, mu) - oracle.dal_cost(p, d, em, I, v, mu)) / (2 * h)
            assert g[m, q] == pytest.approx(fd, rel=2e-5, abs=1e-12), (m, q)


def test_D5_armijo_descent_and_projection():
    rng, I, p, eps = _setup(M=6, seed=9)
    d = oracle.DalParams(M=6, iters=8, sigma0=1e3, b=0.5, c=1e-4, ex_lo=2.0, ex_hi=1100.0, ec_lo=2.0, ec_hi=1100.0)
    eps1, Jh, sh = oracle.dal(p, d, eps, I)
    assert np.all(np.diff(Jh) <= 1e-15)
    assert Jh[-1] < Jh[0]
    assert np.all((eps1[:, 0] >= 2.0) & (eps1[:, 0] <= 1100.0) & (eps1[:, 1] >= 2.0) & (eps1[:, 1] <= 1100.0))
    # replay: each accepted step passes the Armijo test of Algorithm 1 (descent along -D, R25)
    e = eps.copy()
    for it in range(d.iters):
        J0, D = oracle.dal_gradient(p, d, e, I)
        if sh[it] > 0:
            cand = e - sh[it] * D
            cand[:, 0] = np.clip(cand[:, 0], 2.0, 1100.0)
            cand[:, 1] = np.clip(cand[:, 1], 2.0, 1100.0)
            assert oracle.dal_cost(p, d, cand, I) <= J0 - d.c * sh[it] * np.sum(D * D) + 1e-15
            e = cand
    assert np.allclose(e, eps1, rtol=0, atol=1e-12)


def test_dal_admm_multiplier_wiring():
    """Algorithm 2 around DAL (oracle.dal_admm): with gamma = rho the multiplier step
    mu + rho (S_{beta/rho}(grad c - mu/rho) - grad c) equals the projection of mu - rho grad c onto
    the beta-ball per pixel (the Moreau identity, written here as the textbook projection), so after
    one outer iteration from mu = 0, mu = Pi_beta(-rho grad c(T)); and v is the shrink at that c."""
    rng = np.random.default_rng(2)
    H, W, C = 9, 11, 2
    I = rng.random((H, W, C))
    h = 1.0 / (W - 1)
    p = oracle.Params(height=H, width=W, channels=C, radius=9, alpha=0.8 / h, beta=0.7, eps_c=57.0, dt=0.25,
                      rho=0.4, gamma=0.4, iters_per_round=1, rounds=1)
    d = oracle.DalParams(M=5, cost=1, iters=2, sigma0=1e3, ex_lo=8.0)
    eps = np.stack([np.full(5, 40.0), np.full(5, 57.0)], 1)
    e, Jh, c, v, mu = oracle.dal_admm(p, d, eps, I, 1)
    q = oracle.derive(p)
    # independent gradient (forward differences, zero on the last column / row)
    g = np.zeros((H, W, 2 * C))
    g[:, :-1, :C] = (c[:, 1:] - c[:, :-1]) / q.hx
    g[:-1, :, C:] = (c[1:] - c[:-1]) / q.hy
    a = -q.rho * g
    n = np.linalg.norm(a, axis=-1, keepdims=True)
    proj = a * np.minimum(1.0, q.beta / np.maximum(n, 1e-300))
    np.testing.assert_allclose(mu, proj, rtol=1e-12, atol=1e-13)
    assert np.all(np.linalg.norm(mu, axis=-1) <= q.beta * (1 + 1e-12))
    assert np.all(np.diff(Jh[0]) <= 1e-12 * abs(Jh[0][0]))  # Armijo inside


def test_D6_remark34_stopping_rules():
    """Remark 3.4: (a) cost stationarity |J_j - J_{j-1}| / J_{j-1} < eta stops the run at
    the first such j, and the costs up to there are those of the uncapped run (the rule only truncates);
    (b) the projected gradient vanishes identically when E is a single point (every component sits on both
    bounds, so every -D points out of E): the run stops before any step (criterion 2)."""
    rng, I, p, eps = _setup(M=6, seed=9)
    base = dict(M=6, iters=12, sigma0=1e3, b=0.5, c=1e-4)
    _, Jfull, _ = oracle.dal(p, oracle.DalParams(**base), eps, I)
    rel = np.abs(np.diff(Jfull[:-1])) / Jfull[:-2]
    eta = 1e-10  # the paper's tolerance
    assert np.any(rel < eta) and rel[0] >= eta
    first = 1 + int(np.argmax(rel < eta))
    e2, Jh, sh, (run, why) = oracle.dal(p, oracle.DalParams(**base, eta=eta), eps, I, return_stop=True)
    assert why == 1 and run == first, (run, first)
    np.testing.assert_array_equal(Jh[:run], Jfull[:run])
    assert np.all(rel[:run - 1] >= eta) and rel[run - 1] < eta
    # (b) E = {(40, 10)}: projected gradient 0 at the start
    box = dict(ex_lo=40.0, ex_hi=40.0, ec_lo=10.0, ec_hi=10.0)
    e3, Jh3, sh3, (run3, why3) = oracle.dal(p, oracle.DalParams(**base, **box, eta_grad=1e-30), eps, I,
                                           return_stop=True)
    assert (run3, why3) == (0, 2) and len(Jh3) == 1 and len(sh3) == 0
    assert np.all(e3[:, 0] == 40.0) and np.all(e3[:, 1] == 10.0)
    # without the rule the same box runs every iteration (and cannot move)
    _, Jh4, _, (run4, why4) = oracle.dal(p, oracle.DalParams(**base, **box), eps, I, return_stop=True)
    assert (run4, why4) == (12, 0)


def _dual_value_independent(q, c, mu, I):
    """Phi(mu) = min_v L(c, v, mu) = <Huber_{beta,rho}(grad c - mu/rho)> + alpha/2 |c - I|^2 - |mu|^2/(2 rho)
    (eq:complete_square, eq:soft_threshold; reading R27), written out with numpy."""
    H, W, C = c.shape
    g = np.zeros((H, W, 2 * C))
    g[:, :-1, :C] = (c[:, 1:] - c[:, :-1]) / q.hx
    g[:-1, :, C:] = (c[1:] - c[:-1]) / q.hy
    a = g - mu / q.rho
    n = np.linalg.norm(a, axis=-1)
    hub = np.where(n <= q.beta / q.rho, 0.5 * q.rho * n * n, q.beta * n - q.beta ** 2 / (2 * q.rho))
    w = q.hx * q.hy
    return w * (hub.sum() + 0.5 * q.alpha * np.sum((c - I) ** 2) - np.sum(mu * mu) / (2 * q.rho))


def test_D7_gamma_two_way_armijo():
    """The remark after Algorithm 2: the ascent step gamma^(j) by Algorithm 1's
    two-way search on Phi(mu) = min_v L(c(mu), v, mu). Replayed independently: every accepted step passes
    Phi(mu + t g) >= Phi(mu) + c t |g|^2 (Phi by the Huber formula above, not by the oracle's energy_L),
    and the next larger trial t / b fails (the search keeps the last passing step)."""
    rng = np.random.default_rng(4)
    H, W, C = 8, 9, 2
    I = rng.random((H, W, C))
    h = 1.0 / (W - 1)
    p = oracle.Params(height=H, width=W, channels=C, radius=8, alpha=0.8 / h, beta=0.7, eps_c=57.0, dt=0.25,
                      rho=0.4, gamma=0.05, iters_per_round=1, rounds=1)
    d = oracle.DalParams(M=4, cost=1, iters=2, sigma0=1e3, ex_lo=8.0, max_ls=8, b=0.5, c=1e-4)
    eps = np.stack([np.full(4, 40.0), np.full(4, 57.0)], 1)
    q = oracle.derive(p)
    e, Jh, c, v, mu, gh = oracle.dal_admm(p, d, eps, I, 2, gamma_search=True)
    assert np.all(gh > 0)
    # replay the first outer iteration: mu^(0) = 0, v^(-1) = 0
    dq = oracle.DalParams(**{**d.__dict__, "rho": q.rho})
    e0, _, _ = oracle.dal(p, dq, eps, I, np.zeros((H, W, 2 * C)), np.zeros((H, W, 2 * C)))
    _, c0 = oracle.dal_cost(p, dq, e0, I, np.zeros((H, W, 2 * C)), np.zeros((H, W, 2 * C)), return_state=True)
    mu0 = np.zeros((H, W, 2 * C))
    v0 = oracle.shrink_field(p, q.rho, c0, mu0)
    g = v0 - oracle.grad(c0, q.hx, q.hy)
    g2 = q.hx * q.hy * np.sum(g * g)
    phi0 = _dual_value_independent(q, c0, mu0, I)
    assert phi0 == pytest.approx(oracle.dual_value(p, q.rho, c0, mu0, I), rel=1e-12)

    def phi_at(t):
        mt = mu0 + t * g
        et, _, _ = oracle.dal(p, dq, e0, I, v0, mt)
        _, ct = oracle.dal_cost(p, dq, et, I, v0, mt, return_state=True)
        return _dual_value_independent(q, ct, mt, I)

    t = gh[0]
    assert phi_at(t) >= phi0 + d.c * t * g2
    assert phi_at(t / d.b) < phi0 + d.c * (t / d.b) * g2
