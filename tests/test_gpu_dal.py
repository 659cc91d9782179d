"""GPU DAL (msa.h msa_dal / msa_dal_gradient; msa_dal.cu) against the DAL
oracle (pinned by finite differences in tests/test_oracle_dal.py): terminal state, cost and the
discrete-adjoint gradient for both terminal costs, and Algorithm 1's iterates (Armijo descent,
projection onto E, the same accepted steps as the oracle)."""
import numpy as np
import pytest

import oracle
from _harness import hook_env

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")
import os as _os
HERE_DIR = _os.path.dirname(_os.path.abspath(__file__))


def _case(H=16, W=16, C=3, R=15, M=12, seed=0, kernel=0):
    rng = np.random.default_rng(seed)
    blocks = np.repeat(np.repeat(rng.random((4, 4, C)), H // 4, 0), W // 4, 1)
    I = np.clip(blocks + 0.05 * rng.standard_normal((H, W, C)), 0, 1).astype(np.float32)
    h = 1.0 / (W - 1)
    sp = dict(alpha=8.0 / h * 0.1, beta=1.0, radius=R, kernel=kernel, eps_x=0.0, eps_c=57.0, dt=0.25, rho=0.5,
              gamma=0.5, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1, rounds=1)
    eps = np.stack([rng.uniform(30.0, 300.0, M), rng.uniform(20.0, 120.0, M)], axis=1)
    return rng, I, sp, eps


def _oracle_params(I, sp):
    H, W, C = I.shape
    return oracle.Params.from_solver(H, W, C, sp)


@pytest.mark.parametrize("cost,kernel", [(0, 0), (1, 0), (0, 1)])
def test_dal_gradient_parity(cost, kernel):
    rng, I, sp, eps = _case(seed=cost + 2 * kernel, kernel=kernel)
    H, W, C = I.shape
    M = eps.shape[0]
    v = mu = None
    if cost == 1:
        v = (0.3 * rng.standard_normal((H, W, 2 * C))).astype(np.float32)
        mu = (0.3 * rng.standard_normal((H, W, 2 * C))).astype(np.float32)
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
        J, g = s.dal_gradient(msa.DalParams(steps=M, cost=cost), eps, v, mu)
    od = oracle.DalParams(M=M, cost=cost, rho=sp["rho"])
    Jo, go = oracle.dal_gradient(_oracle_params(I, sp), od, eps, I.astype(np.float64), v, mu)
    assert J == pytest.approx(Jo, rel=1e-5)
    scale = np.max(np.abs(go), axis=0)
    err = float(np.max(np.abs(g - go) / scale))
    print(f"dal gradient cost={cost} kernel={kernel}: max |g - g_oracle| / column max = {err:.2e}")
    # The gradient is a sum over M = 12 Euler steps of <lambda^(m+1), dF/deps(c^(m))>: image-wide sums of
    # products of the fp32 adjoint (M transposed-Jacobian stencil steps) with phi' factors. Measured on
    # the B200: 1.4e-7, 2.0e-7 and 8.8e-7 of the column maximum for the three cases (fp32 rounding of
    # the states and addends); the gate keeps about a 10x margin.
    assert err <= 1e-5, err


def test_dal_terminal_state_and_cost():
    rng, I, sp, eps = _case(seed=5, M=20)
    H, W, C = I.shape
    d = msa.DalParams(steps=20, iters=0)
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
        e, Jh, _ = s.dal(d, eps)
        cT = s.get_field(msa.FIELD_C)[0]
    Jo, cTo = oracle.dal_cost(_oracle_params(I, sp), oracle.DalParams(M=20), e, I.astype(np.float64),
                              return_state=True)
    assert Jh[0] == pytest.approx(Jo, rel=1e-5)
    assert np.max(np.abs(cT - cTo)) <= 1e-5


def test_dal_algorithm1_matches_oracle():
    rng, I, sp, eps = _case(seed=7, M=10)
    H, W, C = I.shape
    kw = dict(iters=6, max_ls=25, sigma0=1e4, b=0.5, c=1e-4, ex_lo=2.0, ex_hi=1100.0, ec_lo=2.0, ec_hi=1100.0)
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
        e, Jh, sh = s.dal(msa.DalParams(steps=10, **kw), eps)
    eo, Jho, sho = oracle.dal(_oracle_params(I, sp), oracle.DalParams(M=10, **kw), eps, I.astype(np.float64))
    assert np.all(np.diff(Jh) <= 1e-9 * abs(Jh[0]))      # Armijo: J never increases
    assert Jh[-1] < Jh[0]
    assert np.all((e[:, 0] >= 2.0) & (e[:, 0] <= 1100.0) & (e[:, 1] >= 2.0) & (e[:, 1] <= 1100.0))
    np.testing.assert_allclose(sh, sho, rtol=1e-12)       # same accepted steps
    np.testing.assert_allclose(Jh, Jho, rtol=1e-4)
    np.testing.assert_allclose(e, eo, rtol=2e-3, atol=1e-6)


@pytest.mark.parametrize("R,C,kernel", [(15, 3, 0), (12, 1, 1), (20, 4, 0)])
def test_dal_large_support_kernels_bitwise(R, C, kernel, tmp_path):
    """R > 8 runs the forward and backward steps on the chunked shared-memory kernels; they have the
    generic DAL kernels' arithmetic and summation order: bitwise-equal cost and gradient (with the
    window split of small images switched off; with it, equal to fp32 summation order)."""
    import json
    import os
    import subprocess
    import sys
    script = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
import paper_2510_16154_b200 as msa
spec = json.loads(sys.argv[1])
rng = np.random.default_rng(spec["seed"])
H, W, C, R, M = spec["H"], spec["W"], spec["C"], spec["R"], spec["M"]
I = rng.random((1, H, W, C), dtype=np.float32)
h = 1.0 / (W - 1)
sp = dict(alpha=0.8 / h, beta=1.0, radius=R, kernel=spec["kernel"], eps_x=0.0, eps_c=57.0, dt=0.25, rho=0.5,
          gamma=0.5, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1, rounds=1)
eps = np.stack([rng.uniform(8.0, 200.0, M), rng.uniform(20.0, 120.0, M)], axis=1)
with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I) as s:
    J, g = s.dal_gradient(msa.DalParams(steps=M), eps)
np.savez(sys.argv[2], J=np.array([J]), g=g)
""" % os.path.dirname(HERE_DIR)
    spec = dict(seed=R + C, H=29, W=37, C=C, R=R, M=6, kernel=kernel)
    outs = []
    for variant in ("large", "generic", "large_split"):
        env = hook_env()
        env.pop("MSA_DAL_GENERIC", None)
        env.pop("MSA_LARGE_NOSPLIT", None)
        if variant == "generic":
            env["MSA_DAL_GENERIC"] = "1"
        if variant == "large":  # the window of a pixel in one CTA: the generic order
            env["MSA_LARGE_NOSPLIT"] = "1"
        out = str(tmp_path / f"{variant}.npz")
        subprocess.run([sys.executable, "-c", script, json.dumps(spec), out], check=True, env=env)
        outs.append(np.load(out))
    assert np.array_equal(outs[0]["J"], outs[1]["J"])
    assert np.array_equal(outs[0]["g"], outs[1]["g"])
    # small image: the default splits each window over CTAs (partial sums added in part order) -
    # the same terms in another order
    np.testing.assert_allclose(outs[2]["J"], outs[0]["J"], rtol=1e-6)
    np.testing.assert_allclose(outs[2]["g"], outs[0]["g"], rtol=1e-4, atol=1e-6 * float(np.max(np.abs(outs[0]["g"]))))


@pytest.mark.parametrize("S,R,cost", [(3, 15, 0), (4, 3, 1), (1, 12, 0), (11, 3, 0)])
def test_dal_gradient_checkpointing_bitwise(S, R, cost, tmp_path):
    """Checkpointed adjoint (NEXT-1: the trajectory of M + 1 states does not fit at large images):
    states every S steps, each segment recomputed before its adjoint steps - the same states, so
    the same cost and gradient bit for bit as with the full trajectory (M = 10, ragged last
    segment; S = 1 and S >= M - 1 are the degenerate ends)."""
    import json
    import subprocess
    import sys
    script = r"""
import json, sys, numpy as np
sys.path.insert(0, %r)
import paper_2510_16154_b200 as msa
spec = json.loads(sys.argv[1])
rng = np.random.default_rng(spec["seed"])
H, W, C, R, M = 18, 21, 3, spec["R"], 10
I = rng.random((1, H, W, C), dtype=np.float32)
h = 1.0 / (W - 1)
sp = dict(alpha=0.8 / h, beta=1.0, radius=R, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25, rho=0.5, gamma=0.5,
          kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1, rounds=1)
eps = np.stack([rng.uniform(8.0, 200.0, M), rng.uniform(20.0, 120.0, M)], axis=1)
v = (0.3 * rng.standard_normal((H, W, 2 * C))).astype(np.float32)
mu = (0.3 * rng.standard_normal((H, W, 2 * C))).astype(np.float32)
with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I) as s:
    d = msa.DalParams(steps=M, cost=spec["cost"])
    J, g = s.dal_gradient(d, eps, v if spec["cost"] else None, mu if spec["cost"] else None)
np.savez(sys.argv[2], J=np.array([J]), g=g)
""" % _os.path.dirname(HERE_DIR)
    spec = dict(seed=S + R, R=R, cost=cost)
    outs = []
    for ck in (None, S):
        env = hook_env()
        env.pop("MSA_DAL_CHECKPOINT", None)
        if ck is not None:
            env["MSA_DAL_CHECKPOINT"] = str(ck)
        out = str(tmp_path / f"ck{ck}.npz")
        subprocess.run([sys.executable, "-c", script, json.dumps(spec), out], check=True, env=env)
        outs.append(np.load(out))
    assert np.array_equal(outs[0]["J"], outs[1]["J"])
    assert np.array_equal(outs[0]["g"], outs[1]["g"])


@pytest.mark.parametrize("R,C", [(12, 1), (15, 3)])
def test_dal_admm_matches_oracle(R, C):
    """Algorithm 2 with DAL as line 5 (msa_dal_admm) against oracle.dal_admm: the same accepted DAL
    steps and costs per outer iteration, the optimised controls, and the final multiplier."""
    rng, I, sp, eps = _case(H=16, W=16, C=C, R=R, M=6, seed=R + C)
    sp = dict(sp, rho=0.4, gamma=0.4)
    H, W, _ = I.shape
    kw = dict(iters=3, max_ls=20, sigma0=1e3, b=0.5, c=1e-4, ex_lo=2.0, ex_hi=1100.0, ec_lo=2.0, ec_hi=1100.0)
    outer = 3
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
        e, Jh, recs = s.dal_admm(msa.DalParams(steps=6, cost=1, **kw), eps, outer)
        mu = s.get_field(msa.FIELD_MU)[0]
    eo, Jho, co, vo, muo = oracle.dal_admm(_oracle_params(I, sp), oracle.DalParams(M=6, cost=1, **kw), eps,
                                           I.astype(np.float64), outer)
    assert len(recs) == outer
    np.testing.assert_allclose(Jh, Jho, rtol=1e-4)
    np.testing.assert_allclose(e, eo, rtol=2e-3, atol=1e-6)
    np.testing.assert_allclose(mu, muo, rtol=0, atol=2e-4 * max(1.0, float(np.max(np.abs(muo)))))


def test_dal_stopping_rules_match_oracle():
    """Remark 3.4 on the GPU: with the paper's eta = 1e-10 the run ends at the same
    iteration as the oracle's (cost stationarity), and a one-point box stops it before any step
    (projected gradient, criterion 2)."""
    rng, I, sp, eps = _case(H=16, W=16, C=3, R=15, M=6, seed=21)
    H, W, C = I.shape
    kw = dict(iters=12, max_ls=20, sigma0=1e3, b=0.5, c=1e-4, eta=1e-10)
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
        e, Jh, sh, stop = s.dal(msa.DalParams(steps=6, **kw), eps, return_stop=True)
        e2, Jh2, sh2, stop2 = s.dal(msa.DalParams(steps=6, iters=5, ex_lo=40.0, ex_hi=40.0, ec_lo=10.0, ec_hi=10.0,
                                                  eta_grad=1e-30), eps, return_stop=True)
    eo, Jho, sho, stopo = oracle.dal(_oracle_params(I, sp), oracle.DalParams(M=6, **kw), eps, I.astype(np.float64),
                                     return_stop=True)
    assert stop == stopo, (stop, stopo)
    np.testing.assert_allclose(Jh, Jho, rtol=1e-4)
    assert stop2 == (0, 2) and np.all(e2[:, 0] == 40.0) and np.all(e2[:, 1] == 10.0)


def test_dal_admm_gamma_search_matches_oracle():
    """The remark after Algorithm 2: the ascent step gamma^(j) chosen by the two-way
    Armijo search on Phi(mu) = min_v L(c(mu), v, mu). The GPU (fp32 states, host search) takes the same
    steps as oracle.dal_admm(gamma_search=True) (pinned by tests/test_oracle_dal.py::test_D7) and ends
    at the same multiplier."""
    rng, I, sp, eps = _case(H=16, W=16, C=2, R=12, M=4, seed=33)
    sp = dict(sp, rho=0.4, gamma=0.05)
    H, W, C = I.shape
    kw = dict(iters=2, max_ls=8, sigma0=1e3, b=0.5, c=1e-4, ex_lo=8.0, ex_hi=1100.0, ec_lo=2.0, ec_hi=1100.0)
    outer = 2
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
        e, Jh, recs, gh = s.dal_admm(msa.DalParams(steps=4, cost=1, gamma_ls=1, **kw), eps, outer, return_gamma=True)
        mu = s.get_field(msa.FIELD_MU)[0]
    eo, Jho, co, vo, muo, gho = oracle.dal_admm(_oracle_params(I, sp), oracle.DalParams(M=4, cost=1, **kw), eps,
                                                I.astype(np.float64), outer, gamma_search=True)
    np.testing.assert_array_equal(gh, gho)
    assert np.all(gh > 0)
    np.testing.assert_allclose(Jh, Jho, rtol=1e-4)
    np.testing.assert_allclose(mu, muo, rtol=0, atol=2e-4 * max(1.0, float(np.max(np.abs(muo)))))
