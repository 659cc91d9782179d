"""Regenerates the transcription golden vectors tests/golden/G1_grey_nonsquare.json and
G2_rgb_coupled.json with an independent fp64 NumPy implementation of the SURVEY.md §8(c) oracle block.

It imports neither oracle/ nor the CUDA package: every formula is re-typed here from the definitions of
SURVEY §8.0 and §8(c) (readings R2 window + 1/N_R, R5 node spacing, R6 forward gradient / adjoint
divergence, R7 Chambolle-Pock dual and prox steps, R8 rounds, R21 increment-form prox, R27 Huber), so
the stored vectors pin oracle/msa_oracle.c against a second transcription, not against itself.
The vectors are not the paper's numbers (the paper prints none); they catch transcription slips.

  python tools/golden_numpy.py           # prints both cases as JSON
  tests/test_oracle_pins.py::test_golden_generator_reproduces_stored_vectors runs it (1e-12)
"""
from __future__ import annotations

import json
import math
import sys

import numpy as np


def derive(H, W, R, eps_x=0.0):
    hx = 1.0 / (W - 1) if W > 1 else 1.0
    hy = 1.0 / (H - 1) if H > 1 else 1.0
    if eps_x <= 0:
        eps_x = 2.0 / (R * min(hx, hy)) ** 2  # R2: r >= 1 for |delta| >= R
    L = math.sqrt(4.0 / hx ** 2 + 4.0 / hy ** 2)
    return hx, hy, eps_x, L


def phi(t):  # standard Wendland in t = max(1 - r, 0): t^4 (5 - 4t)  (R3)
    return t ** 4 * (5.0 - 4.0 * t)


def agent_F(c, R, hx, hy, eps_x, eps_c):
    """F(n) = (1/N_R) sum_{delta in D_R, n + delta inside} phi(r) (c(n + delta) - c(n))   (R2)."""
    H, W, C = c.shape
    offs = [(dx, dy) for dy in range(-R, R + 1) for dx in range(-R, R + 1) if dx * dx + dy * dy <= R * R]
    F = np.zeros_like(c)
    for dx, dy in offs:
        if dx == 0 and dy == 0:
            continue
        # neighbour (i + dx, j + dy) of pixel (i, j); row j = 0 is the bottom row (R19)
        j0, j1 = max(0, -dy), min(H, H - dy)
        i0, i1 = max(0, -dx), min(W, W - dx)
        if j0 >= j1 or i0 >= i1:
            continue
        ci = c[j0:j1, i0:i1]
        cj = c[j0 + dy:j1 + dy, i0 + dx:i1 + dx]
        d = cj - ci
        r = 0.5 * eps_x * ((dx * hx) ** 2 + (dy * hy) ** 2) + 0.5 * eps_c * np.sum(d * d, axis=-1)
        w = phi(np.maximum(1.0 - r, 0.0))
        F[j0:j1, i0:i1] += w[..., None] * d
    return F / len(offs)


def grad(u, hx, hy):
    C = u.shape[2]
    g = np.zeros(u.shape[:2] + (2 * C,))
    g[:, :-1, :C] = (u[:, 1:] - u[:, :-1]) / hx
    g[:-1, :, C:] = (u[1:] - u[:-1]) / hy
    return g


def div(p, hx, hy):
    C = p.shape[2] // 2
    px, py = p[..., :C], p[..., C:]
    d = np.zeros(p.shape[:2] + (C,))
    d[:, :-1] += px[:, :-1] / hx
    d[:, 1:] -= px[:, :-1] / hx
    d[:-1] += py[:-1] / hy
    d[1:] -= py[:-1] / hy
    return d


def proj(q, beta):
    n = np.linalg.norm(q, axis=-1, keepdims=True)
    return q * np.minimum(1.0, beta / np.maximum(n, 1e-300))


def run(I, R, eps_x, eps_c, dt, alpha, beta, rho, gamma, K, rounds, theta=1.0, snapshot_after=None):
    H, W, C = I.shape
    hx, hy, ex, L = derive(H, W, R, eps_x)
    tau = sigma = 0.99 / L
    w = hx * hy
    c, cb = I.copy(), I.copy()
    p = np.zeros((H, W, 2 * C))
    mu = np.zeros((H, W, 2 * C))
    snaps, stats = {}, []
    it = 0
    for _ in range(rounds):
        for _ in range(K):
            ch = c + dt * agent_F(c, R, hx, hy, ex, eps_c)                          # step 1
            p = proj((rho * (p + sigma * grad(cb, hx, hy)) - sigma * mu) / (rho + sigma), beta)  # step 2 (R7)
            cn = ch + (tau * div(p, hx, hy) + tau * alpha * (I - ch)) / (1.0 + tau * alpha)  # step 3 (R21)
            cb = cn + theta * (cn - ch)
            c = cn
            it += 1
            if snapshot_after == it:
                snaps["c_after_iteration_1"] = c.copy()
        g = grad(c, hx, hy)
        a = g - mu / rho
        na = np.linalg.norm(a, axis=-1, keepdims=True)
        v = np.maximum(0.0, 1.0 - (beta / rho) / np.maximum(na, 1e-300)) * a        # S_{beta/rho}
        ng = np.linalg.norm(g, axis=-1)
        e_tv = w * beta * ng.sum()
        e_fid = w * 0.5 * alpha * np.sum((c - I) ** 2)
        n = na[..., 0]
        hub = np.where(n <= beta / rho, 0.5 * rho * n * n, beta * n - beta ** 2 / (2 * rho))
        P = w * hub.sum() + e_fid
        dp = div(p, hx, hy)
        D = w * (-np.sum(I * dp) - np.sum(dp * dp) / (2 * alpha) - np.sum(mu * p) / rho - np.sum(p * p) / (2 * rho))
        res = math.sqrt(w * np.sum((v - g) ** 2))
        stats.append({"E_TV": e_tv, "E_fid": e_fid, "P": P, "D": D, "gap": P - D, "residual": res})
        mu = mu + gamma * (v - g)                                                   # Alg. 2 line 7
    return c, mu, stats, snaps, dict(hx=hx, hy=hy, eps_x=ex, L=L, tau=tau)


def G1():
    I = np.array([[0.10, 0.20, 0.80, 0.90], [0.15, 0.25, 0.85, 0.95], [0.10, 0.30, 0.70, 0.90]])[..., None]
    c, mu, st, snaps, dv = run(I, R=2, eps_x=0.0, eps_c=10.0, dt=0.25, alpha=2.0, beta=1.0, rho=0.5, gamma=0.5, K=2,
                               rounds=2, snapshot_after=1)
    return {"c_after_iteration_1": snaps["c_after_iteration_1"][..., 0].tolist(), "c_after_2_rounds": c[..., 0].tolist(),
            "mu_x_after_2_rounds": mu[..., 0].tolist(), "mu_y_after_2_rounds": mu[..., 1].tolist(),
            "round_stats": st, "mean": float(c.mean()), "expect_eps_x": dv["eps_x"], "expect_L": dv["L"],
            "expect_tau": dv["tau"]}


def G2():
    I = np.empty((3, 3, 3))
    I[:, 0:2] = [0.2, 0.4, 0.6]
    I[:, 2] = [0.9, 0.1, 0.3]
    I[1, 1] = [0.25, 0.35, 0.65]
    c, mu, st, _, dv = run(I, R=2, eps_x=2.0, eps_c=57.0, dt=0.25, alpha=3.0, beta=1.0, rho=0.4, gamma=0.4, K=3,
                           rounds=1)
    return {"c_rows_0_and_2": c[0].tolist(), "c_row_1": c[1].tolist(), "round_stats": st,
            "mean": c.reshape(-1, 3).mean(0).tolist(), "expect_tau": dv["tau"], "c_row_2": c[2].tolist()}


if __name__ == "__main__":
    json.dump({"G1": G1(), "G2": G2()}, sys.stdout, indent=1)
    print()
