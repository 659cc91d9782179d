"""Pins of the residual-balancing penalty (oracle.solve_until_balanced):
  RB1  rb_tau = 1 leaves rho fixed: the records equal plain rounds of State.run, bit for bit;
  RB2  the dual residual is rho_r ||div(v_r - v_{r-1})||_w with v_r the round's shrink, re-derived here with
       numpy (shrink S_t(a) = max(0, 1 - t/|a|) a and the forward/adjoint stencils of tools/golden_numpy.py);
  RB3  the rho sequence replays the rule from the recorded primal / dual residuals."""
import os
import sys

import numpy as np
import pytest

import oracle
import synth

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import golden_numpy as gn  # noqa: E402


def _case():
    cfg = synth.resized(synth.CONFIGS["cfg2"], 48, 40, rounds=1, iters_per_round=10)
    img = synth.generate(cfg.recipe)[0].astype(np.float64)
    p = oracle.Params.from_solver(48, 40, 3, synth.solver_params(cfg))
    return p, img


def test_RB1_tau_one_is_plain_rounds():
    p, img = _case()
    st, recs, duals = oracle.solve_until_balanced(p, img, 5, rb_tau=1.0)
    ref = oracle.State(p, img)
    rr = ref.run(5 * p.iters_per_round)
    for a, b in zip(recs, rr):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(st.c, ref.c)


def test_RB2_dual_residual_and_RB3_rule():
    p, img = _case()
    rb_mu, rb_tau = 10.0, 2.0
    st, recs, duals = oracle.solve_until_balanced(p, img, 6, rb_mu=rb_mu, rb_tau=rb_tau)
    q = oracle.derive(p)
    # replay round by round with numpy's shrink and divergence
    s = oracle.State(p, img)
    v_prev = None
    for r in range(6):
        mu_pre, rho_r = s.mu.copy(), s.rho
        s.run(p.iters_per_round)
        g = gn.grad(s.c, q.hx, q.hy)
        a = g - mu_pre / rho_r
        n = np.linalg.norm(a, axis=-1, keepdims=True)
        v = np.maximum(0.0, 1.0 - (q.beta / rho_r) / np.maximum(n, 1e-300)) * a
        if v_prev is None:
            assert np.isnan(duals[r])
        else:
            want = rho_r * np.sqrt(q.hx * q.hy * np.sum(gn.div(v - v_prev, q.hx, q.hy) ** 2))
            assert duals[r] == pytest.approx(want, rel=1e-12)
            prim = recs[r][5]
            if prim > rb_mu * duals[r]:
                s.rho *= rb_tau
            elif duals[r] > rb_mu * prim:
                s.rho /= rb_tau
        assert recs[r][6] == pytest.approx(rho_r, rel=1e-15)  # the record carries the round's rho
        v_prev = v
    np.testing.assert_allclose(s.c, st.c, rtol=0, atol=1e-13)
    rhos = [r[6] for r in recs]
    assert len(set(rhos)) > 1, "the rule should fire on this case"
