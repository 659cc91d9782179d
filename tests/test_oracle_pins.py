"""Pins of the fp64 oracle against what the paper and the mathematics fix (SURVEY.md §8(c)
"What pins each part", P1-P18, plus the golden transcription checks G1/G2). None of these
re-types the oracle's own formula: each pin is a closed form, an invariant, a special case,
an independent solver or brute force."""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def wdot(a, b, hx, hy):
    return hx * hy * float(np.sum(a * b))


# ------------------------------------------------------------------ P1, P2: grad / div
@pytest.mark.parametrize("H,W,C", [(1, 1, 1), (1, 7, 3), (9, 1, 3), (5, 8, 1), (16, 13, 3), (11, 16, 16)])
def test_P1_adjointness(H, W, C):
    """<grad u, p>_w + <u, div p>_w = 0 (exact identity, 1e-12 rel)."""
    rng = np.random.default_rng(H * 100 + W + C)
    u = rng.standard_normal((H, W, C))
    p = rng.standard_normal((H, W, 2 * C))
    hx = 1.0 / (W - 1) if W > 1 else 1.0
    hy = 1.0 / (H - 1) if H > 1 else 1.0
    a = wdot(oracle.grad(u, hx, hy), p, hx, hy)
    b = wdot(u, oracle.div(p, hx, hy), hx, hy)
    scale = hx * hy * (np.sum(np.abs(oracle.grad(u, hx, hy) * p)) + np.sum(np.abs(u * oracle.div(p, hx, hy)))) + 1e-300
    assert abs(a + b) <= 1e-12 * scale


def test_P2_grad_div_special_cases():
    """constant -> 0; u = i h_x on 4x4 -> d_x = 1 except last column, d_y = 0; <1, div p> = 0."""
    hx = hy = 1.0 / 3.0
    const = np.full((4, 4, 2), 0.7)
    assert not np.any(oracle.grad(const, hx, hy))
    u = np.tile((np.arange(4) * hx)[None, :, None], (4, 1, 1))
    g = oracle.grad(u, hx, hy)
    assert np.allclose(g[:, :3, 0], 1.0, atol=1e-14) and np.all(g[:, 3, 0] == 0) and np.all(g[..., 1] == 0)
    rng = np.random.default_rng(3)
    p = rng.standard_normal((6, 5, 4))
    assert abs(np.sum(oracle.div(p, 0.25, 0.2))) <= 1e-12 * np.sum(np.abs(p)) / 0.2


# ------------------------------------------------------------------ P3: closed-form TV
@pytest.mark.parametrize("w,hr,i0,j0,H,W", [(5, 3, 4, 6, 20, 30), (1, 1, 3, 3, 8, 9), (7, 11, 2, 2, 16, 12)])
def test_P3_rectangle_tv_closed_form(w, hr, i0, j0, H, W):
    """E_TV of an isolated rectangle (colour a on b): beta ||a-b|| [(2h_r-1) h_y + (2w-1) h_x + sqrt(h_x^2+h_y^2)]
    (derived from the forward-difference TV of §8.0; SPEC.md:339 is the 2x1 special case)."""
    a, b = np.array([0.9, 0.2, 0.4]), np.array([0.1, 0.3, 0.35])
    u = np.tile(b, (H, W, 1))
    u[j0:j0 + hr, i0:i0 + w] = a
    prm = oracle.Params(height=H, width=W, channels=3, radius=2, alpha=0.0, beta=1.7, rho=1.0, gamma=1.0)
    d = oracle.derive(prm)
    st = oracle.State(prm, u)
    e_tv = st.round_stats()[0]
    expect = 1.7 * np.linalg.norm(a - b) * ((2 * hr - 1) * d.hy + (2 * w - 1) * d.hx + math.hypot(d.hx, d.hy))
    assert e_tv == pytest.approx(expect, rel=1e-13)
    # K of the same field = E_TV + fidelity 0 when I = u
    assert oracle.energy_K(prm, u, u) == pytest.approx(expect, rel=1e-13)


def test_P3_two_pixel_step():
    """TV of the 2x1 step (0, 1): only pixel 0 has a nonzero forward difference."""
    prm = oracle.Params(height=1, width=2, channels=1, alpha=0.0, beta=1.0)
    u = np.array([[[0.0], [1.0]]])
    # h_x = 1, h_y = 1 (size-1 axis): |grad| at pixel 0 = 1, quadrature weight 1
    assert oracle.energy_K(prm, u, u) == pytest.approx(1.0, abs=1e-15)


# ------------------------------------------------------------------ P4, P5, P6: phi, r, F
def test_P4_kernel_values():
    """phi(0)=1, phi(0.5)=0.1875, phi(1)=0; printed phi(0)=-1 (eq:kernel PAPER.md:264)."""
    assert oracle.phi(0.0) == 1.0
    assert oracle.phi(0.5) == pytest.approx(0.1875, abs=1e-16)
    assert oracle.phi(1.0) == 0.0 and oracle.phi(1.5) == 0.0
    assert oracle.phi(0.0, kernel=1) == -1.0
    assert oracle.phi(0.5, kernel=1) == pytest.approx(1.0 * 0.0625, abs=1e-16)
    # C^2 Wendland: phi'(1) = phi''(1) = 0 and phi'(0) = 0 (Wendland 1995), checked by differences
    e = 1e-5
    assert abs((oracle.phi(1.0) - oracle.phi(1.0 - e)) / e) < 1e-8
    assert abs((oracle.phi(e) - oracle.phi(0.0)) / e) < 1e-3


def test_P5_pair_distance():
    """r = eps_x/2 |dx|^2 + eps_c/2 dc^2 (eq:ellipsoid)."""
    assert oracle.pair_r(0.3, 0.4, 0.2, 0.0, 0.0) == 0.0
    assert oracle.pair_r(1.0, 0.0, 0.0, 2.0, 5.0) == 1.0
    assert oracle.pair_r(0.6, 0.8, 0.0, 2.0, 0.0) == pytest.approx(1.0, abs=1e-15)
    assert oracle.pair_r(0.0, 0.0, 0.25, 0.0, 8.0) == 1.0


def test_P6_two_agent_rhs():
    """2x1 grey image (0, 1): F = (w/N_R, -w/N_R), w = phi(r) (SPEC.md:175-177 with 1/N -> 1/N_R)."""
    prm = oracle.Params(height=1, width=2, channels=1, radius=2, eps_x=0.2, eps_c=0.4)
    c = np.array([[[0.0], [1.0]]])
    F = oracle.agent_rhs(prm, c)
    r = 0.5 * 0.2 * 1.0 + 0.5 * 0.4 * 1.0  # h_x = 1
    w = (4 * r + 1) * (1 - r) ** 4
    assert F[0, 0, 0] == pytest.approx(w / 13, rel=1e-14)
    assert F[0, 1, 0] == pytest.approx(-w / 13, rel=1e-14)
    # uniform field -> 0; colour far apart (no pair interacts) -> 0
    prm_u = oracle.Params(height=3, width=4, channels=2, radius=2, eps_x=0.2, eps_c=0.4)
    assert not np.any(oracle.agent_rhs(prm_u, np.full((3, 4, 2), 0.3)))
    prm2 = oracle.Params(height=1, width=2, channels=1, radius=2, eps_x=0.2, eps_c=400.0)
    assert not np.any(oracle.agent_rhs(prm2, c))


# ------------------------------------------------------------------ P7: window == paper's full sum
@pytest.mark.parametrize("H,W,C,R", [(16, 16, 3, 3), (9, 14, 1, 2), (12, 10, 16, 5)])
def test_P7_window_equals_all_pairs(H, W, C, R):
    """N_R F_build(n) = sum_j phi(r_ij)(c_j - c_i) over ALL pixels j (eq:MAsystem PAPER.md:91 without 1/N)
    whenever eps_x >= 2/(R h)^2, i.e. supp phi lies inside D_R (reading R2). Brute force."""
    rng = np.random.default_rng(H + W + C + R)
    c = rng.random((H, W, C))
    hx, hy = 1.0 / (W - 1), 1.0 / (H - 1)
    eps_x = 2.0 / (R * min(hx, hy)) ** 2 * (1.0 + rng.random())
    eps_c = 3.0
    prm = oracle.Params(height=H, width=W, channels=C, radius=R, eps_x=eps_x, eps_c=eps_c)
    F = oracle.agent_rhs(prm, c)
    NR = oracle.window_size(R)
    ys, xs = np.meshgrid(np.arange(H) * hy, np.arange(W) * hx, indexing="ij")
    pos = np.stack([xs.ravel(), ys.ravel()], 1)
    col = c.reshape(-1, C)
    dpos2 = np.sum((pos[None, :, :] - pos[:, None, :]) ** 2, -1)
    dcol = col[None, :, :] - col[:, None, :]
    r = eps_x / 2 * dpos2 + eps_c / 2 * np.sum(dcol ** 2, -1)
    phi = np.where(r <= 1.0, (4 * r + 1) * np.clip(1 - r, 0, None) ** 4, 0.0)
    full = np.einsum("ij,ijk->ik", phi, dcol).reshape(H, W, C)
    assert np.max(np.abs(NR * F - full)) <= 1e-14 * max(1.0, np.max(np.abs(full)))


# ------------------------------------------------------------------ P8, P9: invariants
def _rand_params(H, W, C, **kw):
    base = dict(height=H, width=W, channels=C, radius=2, eps_c=57.0, dt=0.25, alpha=8.0 * (W - 1), beta=1.0,
                rho=2.5 / (W - 1), gamma=2.5 / (W - 1), iters_per_round=10, rounds=3)
    base.update(kw)
    return oracle.Params(**base)


@pytest.mark.parametrize("alpha_scale,beta", [(0.0, 0.0), (1.0, 1.0)])
def test_P8_mean_preserved(alpha_scale, beta):
    """Per-channel mean preserved: pure eq:MAsystem (alpha = beta = 0, zero control) by antisymmetry,
    and the whole iteration for any alpha, beta >= 0 since sum div = 0 and c0 = I."""
    rng = np.random.default_rng(11)
    I = rng.random((14, 17, 3))
    prm = _rand_params(14, 17, 3, alpha=8.0 * 16 * alpha_scale, beta=beta, eps_c=5.0, radius=3)
    s = oracle.State(prm, I)
    s.run(100)
    assert np.allclose(s.c.reshape(-1, 3).mean(0), I.reshape(-1, 3).mean(0), rtol=1e-12, atol=0)


def test_P9_constant_image_fixed_point_bitwise():
    """I constant => c = cbar = I, p = mu = 0 bitwise, every iteration (Alg. 2 algebra + R21)."""
    I = np.tile(np.array([0.25, 0.5, 0.875]), (9, 11, 1))
    s = oracle.State(_rand_params(9, 11, 3), I)
    for _ in range(5):
        s.run(7)
        assert np.array_equal(s.c, I) and np.array_equal(s.cbar, I)
        assert not np.any(s.p) and not np.any(s.mu)


# ------------------------------------------------------------------ P10, P11: step 1
def test_P10_maximum_principle():
    """Standard phi, dt <= 1: min c <= c_half <= max c per channel (dt sum phi / N_R < 1)."""
    rng = np.random.default_rng(5)
    for trial in range(5):
        c = rng.random((12, 13, 3))
        prm = oracle.Params(height=12, width=13, channels=3, radius=3, eps_x=float(rng.uniform(1, 400)),
                            eps_c=float(rng.uniform(0, 60)), dt=1.0)
        ch = c + 1.0 * oracle.agent_rhs(prm, c)
        for k in range(3):
            assert ch[..., k].min() >= c[..., k].min() - 1e-15 and ch[..., k].max() <= c[..., k].max() + 1e-15


def test_P11_cosine_eigenfunction():
    """C=1, eps_c=0, c = cos(w i): away from the border c_half = (1 + dt m(w)) c with
    m(w) = (1/N_R) sum_{delta in D_R} phi(eps_x/2 |delta|_h^2)(cos(w delta_x) - 1) (linear stencil symbol)."""
    H, W, R, om = 15, 40, 3, 0.7
    hx, hy = 1.0 / (W - 1), 1.0 / (H - 1)
    eps_x = 2.0 / (R * min(hx, hy)) ** 2 * 0.6  # some pairs inside the ring are cut by phi
    prm = oracle.Params(height=H, width=W, channels=1, radius=R, eps_x=eps_x, eps_c=0.0, dt=0.25)
    c = np.tile(np.cos(om * np.arange(W))[None, :, None], (H, 1, 1))
    ch = c + 0.25 * oracle.agent_rhs(prm, c)
    m = 0.0
    NR = 0
    for dy in range(-R, R + 1):
        for dx in range(-R, R + 1):
            if dx * dx + dy * dy <= R * R:
                NR += 1
                r = eps_x / 2 * ((dx * hx) ** 2 + (dy * hy) ** 2)
                m += ((4 * r + 1) * (1 - r) ** 4 if r < 1 else 0.0) * (math.cos(om * dx) - 1)
    m /= NR
    inner = ch[R:H - R, R:W - R, 0]
    assert np.max(np.abs(inner - (1 + 0.25 * m) * c[R:H - R, R:W - R, 0])) <= 1e-15


# ------------------------------------------------------------------ P12: shrink / projection
def _shrink(a: np.ndarray, rho: float, beta: float = 1.0) -> np.ndarray:
    """v = S_{beta/rho}(a) through the oracle (c = 0 so grad c = 0, mu = -rho a)."""
    H, W, C2 = a.shape
    prm = oracle.Params(height=H, width=W, channels=C2 // 2, beta=beta, rho=rho, gamma=rho)
    return oracle.shrink_field(prm, rho, np.zeros((H, W, C2 // 2)), -rho * a)


def test_P12_shrink_examples_and_optimality():
    """eq:soft_threshold PAPER.md:431-440: |a| <= 1/rho -> 0; (2,0), rho=1 -> (1,0);
    v minimises f(v) = rho/2 |v-a|^2 + |v| (grid search); Moreau S_t(a) = a - Pi_t(a)."""
    v = _shrink(np.array([[[2.0, 0.0]]]), 1.0)
    assert np.allclose(v[0, 0], [1.0, 0.0], atol=1e-15)
    assert not np.any(_shrink(np.array([[[0.3, -0.4]]]), 2.0))  # |a| = 0.5 <= 1/2
    rng = np.random.default_rng(9)
    for _ in range(20):
        a = rng.standard_normal(2) * 1.5
        rho = float(rng.uniform(0.3, 3.0))
        vs = _shrink(a[None, None, :], rho)[0, 0]
        f = lambda v: rho / 2 * np.sum((v - a) ** 2) + np.linalg.norm(v)
        grid = np.linspace(-4, 4, 321)
        gv = np.stack(np.meshgrid(grid, grid, indexing="ij"), -1).reshape(-1, 2)
        fg = rho / 2 * np.sum((gv - a) ** 2, 1) + np.linalg.norm(gv, axis=1)
        assert f(vs) <= fg.min() + 1e-12
        t = 1.0 / rho
        proj = a * min(1.0, t / np.linalg.norm(a))
        assert np.allclose(vs, a - proj, atol=1e-14)


def test_P12_gamma_equals_rho_collapse():
    """At gamma = rho: mu + rho (S_{beta/rho}(g - mu/rho) - g) = Pi_beta(mu - rho g) (identity)."""
    rng = np.random.default_rng(21)
    H, W, C = 6, 7, 3
    c = rng.random((H, W, C))
    mu = rng.standard_normal((H, W, 2 * C))
    rho, beta = 0.37, 1.3
    prm = oracle.Params(height=H, width=W, channels=C, beta=beta, rho=rho, gamma=rho)
    s = oracle.State(prm, c)
    s.c[...] = c
    s.mu[...] = mu
    s.rho = rho
    s.round_update()
    d = oracle.derive(prm)
    q = mu - rho * oracle.grad(c, d.hx, d.hy)
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    expect = q * np.minimum(1.0, beta / np.maximum(n, 1e-300))
    assert np.max(np.abs(s.mu - expect)) <= 1e-13


# ------------------------------------------------------------------ P13: complete square, P = min_v L~
def test_P13_complete_square_identity():
    """L~(u,v) = L(u,v,mu) + int |mu|^2/(2 rho) (eq:complete_square PAPER.md:399-403), and the round's
    primal value P equals L~(u, S(grad u - mu/rho)) (the v-minimum, eq:soft_threshold)."""
    rng = np.random.default_rng(4)
    H, W, C = 8, 9, 3
    u, I = rng.random((H, W, C)), rng.random((H, W, C))
    v, mu = rng.standard_normal((H, W, 2 * C)), rng.standard_normal((H, W, 2 * C))
    rho = 0.8
    prm = oracle.Params(height=H, width=W, channels=C, alpha=3.0, beta=1.2, rho=rho, gamma=rho)
    d = oracle.derive(prm)
    Lt = oracle.energy_Ltilde(prm, rho, u, v, mu, I)
    L = oracle.energy_L(prm, rho, u, v, mu, I)
    assert Lt - L - d.hx * d.hy * np.sum(mu * mu) / (2 * rho) == pytest.approx(0.0, abs=1e-12 * abs(Lt))
    s = oracle.State(prm, I)
    s.c[...] = u
    s.mu[...] = mu
    P = s.round_stats()[2]
    vstar = oracle.shrink_field(prm, rho, u, mu)
    assert P == pytest.approx(oracle.energy_Ltilde(prm, rho, u, vstar, mu, I), rel=1e-12)
    # and v* is the minimiser: random perturbations do not decrease L~
    for _ in range(50):
        dv = rng.standard_normal(v.shape) * 1e-3
        assert oracle.energy_Ltilde(prm, rho, u, vstar + dv, mu, I) >= P - 1e-14


# ------------------------------------------------------------------ P14, P15: duality, monotonicity (dt = 0)
def test_P14_P15_gap_and_monotonicity_tiny_case():
    """dt = 0 (pure CP on L~ with v eliminated, R7): weak duality gap >= 0 at every iterate (Thm 4.2
    PAPER.md:363-382, discrete analogue); ||z^{k+1}-z^k||_M non-increasing within a round (CP is a proximal
    point method in M = [[I/tau, -grad^T], [-grad, I/sigma]]); gap non-increasing within a round and AL
    residual decreasing across rounds (north_star, the tiny case)."""
    rng = np.random.default_rng(12)
    H, W, C = 12, 12, 3
    I = rng.random((H, W, C))
    h = 1.0 / (W - 1)
    prm = oracle.Params(height=H, width=W, channels=C, radius=2, dt=0.0, alpha=8.0 / h, beta=1.0, rho=2.5 * h,
                        gamma=2.5 * h, iters_per_round=60, rounds=4)
    d = oracle.derive(prm)
    s = oracle.State(prm, I)
    res = []
    for r in range(4):
        gaps, mnorm = [], []
        prev_c, prev_p = s.c.copy(), s.p.copy()
        for k in range(60):
            s.iteration()
            st = s.round_stats()
            gaps.append(st[4])
            du, dp = s.c - prev_c, s.p - prev_p
            m2 = np.sum(du * du) / d.tau - 2 * np.sum(oracle.grad(du, d.hx, d.hy) * dp) + np.sum(dp * dp) / d.sigma
            mnorm.append(m2)
            prev_c, prev_p = s.c.copy(), s.p.copy()
        assert min(gaps) >= -1e-12
        assert all(mnorm[k + 1] <= mnorm[k] * (1 + 1e-9) + 1e-25 for k in range(len(mnorm) - 1))
        assert all(gaps[k + 1] <= gaps[k] + 1e-12 for k in range(len(gaps) - 1))
        res.append(s.round_stats()[5])
        s.round_update()
    assert all(res[r + 1] < res[r] for r in range(len(res) - 1))


# ------------------------------------------------------------------ P16: alpha limits
def test_P16_alpha_limits():
    """alpha -> inf gives I, alpha -> 0 gives a constant image, dt = 0."""
    rng = np.random.default_rng(16)
    I = rng.random((8, 8, 3))
    h = 1.0 / 7
    big = oracle.Params(height=8, width=8, channels=3, dt=0.0, alpha=1e12 / h, beta=1.0, rho=2.5 * h, gamma=2.5 * h,
                        iters_per_round=50, rounds=2)
    s = oracle.solve(big, I)
    assert np.max(np.abs(s.c - I)) <= 1e-9
    small = oracle.Params(height=8, width=8, channels=3, dt=0.0, alpha=1e-6 / h, beta=1.0, rho=2.5 * h,
                          gamma=2.5 * h, iters_per_round=200, rounds=60)
    s = oracle.solve(small, I)
    spread = np.max(s.c.reshape(-1, 3).max(0) - s.c.reshape(-1, 3).min(0))
    assert spread <= 1e-6
    assert np.allclose(s.c.reshape(-1, 3).mean(0), I.reshape(-1, 3).mean(0), atol=1e-12)


# ------------------------------------------------------------------ P17: brute force on 8x8
def _np_grad(u, hx, hy):
    g = np.zeros(u.shape[:2] + (2 * u.shape[2],))
    C = u.shape[2]
    g[:, :-1, :C] = (u[:, 1:] - u[:, :-1]) / hx
    g[:-1, :, C:] = (u[1:] - u[:-1]) / hy
    return g


def _np_div(p, hx, hy):
    C = p.shape[2] // 2
    px, py = p[..., :C], p[..., C:]
    d = np.zeros(p.shape[:2] + (C,))
    d[:, :-1] += px[:, :-1] / hx
    d[:, 1:] -= px[:, :-1] / hx
    d[:-1, :] += py[:-1] / hy
    d[1:, :] -= py[:-1] / hy
    return d


def _naive_energies(u, v, mu, I, p, alpha, beta, rho, hx, hy):
    """Pure-Python loops over pixels (independent evaluation of K, L, L~, P, D on a small grid)."""
    H, W, C = u.shape
    g = _np_grad(u, hx, hy)
    dp = _np_div(p, hx, hy)
    K = Lv = Lt = P = Dv = 0.0
    for j in range(H):
        for i in range(W):
            gn = math.sqrt(sum(g[j, i, m] ** 2 for m in range(2 * C)))
            fid = sum((u[j, i, k] - I[j, i, k]) ** 2 for k in range(C)) * alpha / 2
            K += beta * gn + fid
            vn = math.sqrt(sum(v[j, i, m] ** 2 for m in range(2 * C)))
            Lv += beta * vn + fid + sum(mu[j, i, m] * (v[j, i, m] - g[j, i, m]) +
                                        rho / 2 * (v[j, i, m] - g[j, i, m]) ** 2 for m in range(2 * C))
            Lt += beta * vn + fid + rho / 2 * sum((v[j, i, m] - g[j, i, m] + mu[j, i, m] / rho) ** 2
                                                  for m in range(2 * C))
            a = [g[j, i, m] - mu[j, i, m] / rho for m in range(2 * C)]
            na = math.sqrt(sum(x * x for x in a))
            P += (rho * na * na / 2 if na <= beta / rho else beta * na - beta * beta / (2 * rho)) + fid
            Dv += -sum(I[j, i, k] * dp[j, i, k] + dp[j, i, k] ** 2 / (2 * alpha) for k in range(C)) - sum(
                mu[j, i, m] * p[j, i, m] / rho + p[j, i, m] ** 2 / (2 * rho) for m in range(2 * C))
    w = hx * hy
    return w * K, w * Lv, w * Lt, w * P, w * Dv


def test_P17i_brute_force_energies():
    rng = np.random.default_rng(17)
    H = W = 8
    C = 3
    u, I = rng.random((H, W, C)), rng.random((H, W, C))
    v, mu, p = (rng.standard_normal((H, W, 2 * C)) for _ in range(3))
    alpha, beta, rho = 5.0, 0.9, 0.6
    prm = oracle.Params(height=H, width=W, channels=C, alpha=alpha, beta=beta, rho=rho, gamma=rho)
    d = oracle.derive(prm)
    K, Lv, Lt, P, D = _naive_energies(u, v, mu, I, p, alpha, beta, rho, d.hx, d.hy)
    assert oracle.energy_K(prm, u, I) == pytest.approx(K, rel=1e-12)
    assert oracle.energy_L(prm, rho, u, v, mu, I) == pytest.approx(Lv, rel=1e-12)
    assert oracle.energy_Ltilde(prm, rho, u, v, mu, I) == pytest.approx(Lt, rel=1e-12)
    s = oracle.State(prm, I)
    s.c[...] = u
    s.mu[...] = mu
    s.p[...] = p
    st = s.round_stats()
    assert st[2] == pytest.approx(P, rel=1e-12)
    assert st[3] == pytest.approx(D, rel=1e-12)


def _chambolle_rof(I, alpha, beta, hx, hy, iters=200000):
    """Independent ROF solver (dual projection): u = I + div p/alpha, p <- Pi_beta(p + s grad u), s < 2 alpha/L^2."""
    p = np.zeros(I.shape[:2] + (2 * I.shape[2],))
    L2 = 4 / hx ** 2 + 4 / hy ** 2
    s = 1.9 * alpha / L2
    for _ in range(iters):
        u = I + _np_div(p, hx, hy) / alpha
        q = p + s * _np_grad(u, hx, hy)
        n = np.linalg.norm(q, axis=-1, keepdims=True)
        p_new = q * np.minimum(1.0, beta / np.maximum(n, 1e-300))
        if np.max(np.abs(p_new - p)) < 1e-15:
            p = p_new
            break
        p = p_new
    return I + _np_div(p, hx, hy) / alpha


def test_P17ii_dt0_reaches_rof_minimiser():
    """dt = 0: the multiplier rounds remove the Huber bias; c minimises K (eq:cost_TV) and matches an
    independent fp64 ROF solver within 1e-6."""
    rng = np.random.default_rng(170)
    H = W = 8
    C = 3
    I = rng.random((H, W, C))
    h = 1.0 / 7
    prm = oracle.Params(height=H, width=W, channels=C, radius=2, dt=0.0, alpha=8.0 / h * 0.3, beta=1.0,
                        rho=2.5 * h * 40, gamma=2.5 * h * 40, iters_per_round=200, rounds=200)
    s = oracle.solve(prm, I)
    assert s.stats[-1][5] <= 1e-10  # AL residual: the multiplier method has converged
    d = oracle.derive(prm)
    ref = _chambolle_rof(I, prm.alpha, prm.beta, d.hx, d.hy)
    assert np.max(np.abs(s.c - ref)) <= 1e-9
    K0 = oracle.energy_K(prm, s.c, I)
    for _ in range(2000):
        dvec = rng.standard_normal(I.shape)
        dvec /= np.linalg.norm(dvec)
        for step in (1e-2, -1e-2, 1e-3, -1e-3):
            assert oracle.energy_K(prm, s.c + step * dvec, I) >= K0 - 1e-12


# ------------------------------------------------------------------ P18: labels
def _sort_and_gap_count(values: np.ndarray, delta: float) -> int:
    """SPEC.md:568-576's grey-scale rule: sort, open a new cluster at every gap > delta."""
    v = np.sort(values.ravel())
    return 1 + int(np.sum(np.diff(v) > delta))


def test_P18_labels_piecewise_constant():
    rng = np.random.default_rng(18)
    levels = np.array([0.05, 0.21, 0.44, 0.6, 0.93])
    H, W = 20, 23
    lab = rng.integers(0, 5, size=(H, W))
    c = levels[lab][..., None].astype(np.float32)
    out, n, pal = oracle.labels(c, 0.1, max_k=8)
    assert n == _sort_and_gap_count(c, 0.1) == 5
    # count invariant under a pixel permutation; labels canonical (first appearance order)
    perm = rng.permutation(H * W)
    out2, n2, _ = oracle.labels(c.reshape(-1, 1)[perm].reshape(H, W, 1), 0.1)
    assert n2 == n
    first = {}
    for idx, l in enumerate(out.ravel()):
        first.setdefault(l, idx)
    assert [first[k] for k in range(n)] == sorted(first.values())
    # same cluster <=> same level
    for a in range(5):
        assert len(np.unique(out[lab == a])) == 1
    # perturbations smaller than margin/2 change nothing (margin = min level gap - delta)
    margin = np.min(np.diff(levels)) - 0.1
    noisy = (c + rng.uniform(-margin / 4, margin / 4, c.shape)).astype(np.float32)
    out3, n3, _ = oracle.labels(noisy, 0.1)
    assert n3 == n and np.array_equal(out3, out)
    assert np.allclose(np.sort(pal[:, 0]), levels, atol=1e-6)


def test_P18_labels_brute_force_union_find():
    """Stage (i)+(ii) against a brute-force transitive closure on a tiny RGB field."""
    rng = np.random.default_rng(181)
    H, W, C, delta = 6, 7, 3, 0.15
    c = (rng.integers(0, 4, (H, W, C)) * 0.12 + rng.uniform(0, 0.02, (H, W, C))).astype(np.float32)
    lab, n, _ = oracle.labels(c, delta)
    N = H * W
    flat = c.reshape(N, C)
    adj = np.zeros((N, N), bool)
    for j in range(H):
        for i in range(W):
            a = j * W + i
            for b in ([a + 1] if i + 1 < W else []) + ([a + W] if j + 1 < H else []):
                if np.all(np.abs(flat[a] - flat[b]) <= np.float32(delta)):
                    adj[a, b] = adj[b, a] = True
    seg = np.arange(N)
    changed = True
    while changed:
        changed = False
        for a in range(N):
            for b in np.nonzero(adj[a])[0]:
                m = min(seg[a], seg[b])
                if seg[a] != m or seg[b] != m:
                    seg[a] = seg[b] = m
                    changed = True
    segs = sorted(set(seg))
    means = {s: np.round(flat[seg == s].astype(np.float64) * 2 ** 32).sum(0) / np.sum(seg == s) * 2 ** -32
             for s in segs}
    cl = {s: s for s in segs}
    changed = True
    while changed:
        changed = False
        for s in segs:
            for t in segs:
                if cl[s] != cl[t] and np.all(np.abs(means[s] - means[t]) <= delta):
                    m = min(cl[s], cl[t])
                    for q in segs:
                        if cl[q] in (cl[s], cl[t]):
                            cl[q] = m
                    changed = True
    roots = sorted(set(cl.values()))
    expect = np.array([roots.index(cl[seg[a]]) for a in range(N)]).reshape(H, W)
    assert n == len(roots)
    assert np.array_equal(lab, expect)


# ------------------------------------------------------------------ golden transcription checks
def test_G1_golden():
    g = json.load(open(os.path.join(GOLDEN, "G1_grey_nonsquare.json")))
    I = np.array(g["input_rows_bottom_to_top"])[..., None]
    gp = g["params"]
    prm = oracle.Params(height=3, width=4, channels=1, radius=gp["radius"], eps_c=gp["eps_c"], dt=gp["dt"],
                        alpha=gp["alpha"], beta=gp["beta"], rho=gp["rho"], gamma=gp["gamma"],
                        iters_per_round=gp["iters_per_round"], rounds=gp["rounds"])
    d = oracle.derive(prm)
    assert d.eps_x == pytest.approx(gp["expect_eps_x"], rel=1e-15)
    assert d.tau == pytest.approx(gp["expect_tau"], rel=1e-15)
    s = oracle.State(prm, I)
    s.run(1)
    assert np.max(np.abs(s.c[..., 0] - np.array(g["c_after_iteration_1"]))) <= 1e-12
    s.run(3)
    assert np.max(np.abs(s.c[..., 0] - np.array(g["c_after_2_rounds"]))) <= 1e-12
    assert np.max(np.abs(s.mu[..., 0] - np.array(g["mu_x_after_2_rounds"]))) <= 1e-12
    assert np.max(np.abs(s.mu[..., 1] - np.array(g["mu_y_after_2_rounds"]))) <= 1e-12
    for st, ref in zip(s.stats, g["round_stats"]):
        for idx, key in enumerate(["E_TV", "E_fid", "P", "D", "gap", "residual"]):
            assert st[idx] == pytest.approx(ref[key], rel=1e-12, abs=1e-14)
        assert st[8] == pytest.approx(g["mean"], rel=1e-13)


def test_G2_golden():
    g = json.load(open(os.path.join(GOLDEN, "G2_rgb_coupled.json")))
    I = np.tile(np.array(g["colour_cols_0_1"]), (3, 3, 1))
    I[:, 2] = g["colour_col_2"]
    I[1, 1] = g["centre_pixel_1_1"]
    gp = g["params"]
    prm = oracle.Params(height=3, width=3, channels=3, radius=gp["radius"], eps_x=gp["eps_x"], eps_c=gp["eps_c"],
                        dt=gp["dt"], alpha=gp["alpha"], beta=gp["beta"], rho=gp["rho"], gamma=gp["gamma"],
                        iters_per_round=gp["iters_per_round"], rounds=gp["rounds"])
    assert oracle.derive(prm).tau == pytest.approx(gp["expect_tau"], rel=1e-15)
    s = oracle.solve(prm, I)
    assert np.max(np.abs(s.c[0] - np.array(g["c_rows_0_and_2"]))) <= 1e-12
    assert np.max(np.abs(s.c[2] - np.array(g["c_rows_0_and_2"]))) <= 1e-12
    assert np.max(np.abs(s.c[1] - np.array(g["c_row_1"]))) <= 1e-12
    st, ref = s.stats[0], g["round_stats"][0]
    for idx, key in enumerate(["E_TV", "E_fid", "P", "D", "gap", "residual"]):
        assert st[idx] == pytest.approx(ref[key], rel=1e-12)
    assert np.allclose(st[8:11], g["mean"], atol=1e-15)


# ------------------------------------------------------------------ crop locality (sampled full-size parity)
def test_crop_locality_exact():
    """The oracle run on a crop with the full image's spacing reproduces the full run bitwise on pixels at least
    n_iters * reach from the crop's artificial edges (basis of the sampled full-size GPU parity checks)."""
    rng = np.random.default_rng(77)
    H, W, C, R, n = 40, 44, 3, 3, 2
    I = rng.random((H, W, C))
    base = dict(channels=C, radius=R, eps_c=57.0, dt=0.25, alpha=8.0 * (W - 1), beta=1.0, rho=2.5 / (W - 1),
                gamma=2.5 / (W - 1), iters_per_round=1000, rounds=1)
    full = oracle.State(oracle.Params(height=H, width=W, **base), I)
    full.run(n)
    reach = R + 2
    j0, j1, i0, i1 = 10, 30, 0, 25  # touches the real left border
    m = n * reach
    cj0, cj1, ci0, ci1 = max(0, j0 - m), min(H, j1 + m), max(0, i0 - m), min(W, i1 + m)
    crop = oracle.State(oracle.Params(height=cj1 - cj0, width=ci1 - ci0, hx=1.0 / (W - 1), hy=1.0 / (H - 1),
                                      **base), I[cj0:cj1, ci0:ci1])
    crop.run(n)
    assert np.array_equal(crop.c[j0 - cj0:j1 - cj0, i0 - ci0:i1 - ci0], full.c[j0:j1, i0:i1])


def test_golden_generator_reproduces_stored_vectors():
    """Provenance of G1/G2: the committed independent NumPy transcription of the §8(c) block
    (tools/golden_numpy.py, which imports neither oracle/ nor the CUDA package) regenerates every stored
    value to 1e-12."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), "..", "tools"))
    import golden_numpy as gn
    g1 = json.load(open(os.path.join(GOLDEN, "G1_grey_nonsquare.json")))
    g2 = json.load(open(os.path.join(GOLDEN, "G2_rgb_coupled.json")))
    a, b = gn.G1(), gn.G2()
    for k in ("c_after_iteration_1", "c_after_2_rounds", "mu_x_after_2_rounds", "mu_y_after_2_rounds"):
        np.testing.assert_allclose(np.array(a[k], float), np.array(g1[k], float), rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.array(b["c_rows_0_and_2"]), np.array(g2["c_rows_0_and_2"]), rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.array(b["c_row_2"]), np.array(g2["c_rows_0_and_2"]), rtol=0, atol=1e-12)
    np.testing.assert_allclose(np.array(b["c_row_1"]), np.array(g2["c_row_1"]), rtol=0, atol=1e-12)
    for got, want in ((a["round_stats"], g1["round_stats"]), (b["round_stats"], g2["round_stats"])):
        for r, rec in enumerate(want):
            for k, v in rec.items():
                assert abs(got[r][k] - v) <= 1e-12 * max(1.0, abs(v)), (r, k)
    assert a["expect_tau"] == pytest.approx(g1["params"]["expect_tau"], rel=1e-15)
    assert b["expect_tau"] == pytest.approx(g2["params"]["expect_tau"], rel=1e-15)
