"""GPU parity of the single-loop linearised ADMM scheme (msa.h MSA_SCHEME_LINEARISED_ADMM,
SURVEY §8(f) NEXT-2) against the oracle (oracle/msa_oracle.c mo_iteration_lin, pinned in
tests/test_oracle_lin.py): the BASELINE recipes at reduced size with their full iteration
counts - c within 1e-4 per pixel (R17), labels >= 99.9 % with the same count, round records
(ROF primal, dual of p = -mu, gap, residual) within 1e-3; one step from a random state; the
constant image; the interior/boundary split of rows mode."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from _harness import config_case, rel_err_per_pixel, run_oracle, hook_env

pytestmark = pytest.mark.gpu

msa = pytest.importorskip("paper_2510_16154_b200")
LIN = 1


def _sp(sp):
    return dict(sp, scheme=LIN, tau=0.0, kappa=min(sp["kappa"], 1.0))


@pytest.mark.parametrize("case", [("cfg1", None, None, None), ("cfg2", 96, 80, None), ("cfg3", 64, 72, None),
                                  ("cfg4", 70, 64, None), ("cfg5", 40, 48, 2)])
def test_lin_config_parity(case):
    name, H, W, B = case
    cfg, img, sp = config_case(name, H, W, B)
    sp = _sp(sp)
    Bn, Hh, Ww, C = img.shape
    with msa.Solver(msa.Params.from_solver(Bn, Hh, Ww, C, sp), img) as s:
        gst = s.solve()
        gc = s.get_field(msa.FIELD_C)
        gmu = s.get_field(msa.FIELD_MU)
        glab, gcnt, _ = s.labels(cfg.delta_label)
    refs = run_oracle(img, sp)
    for b, o in enumerate(refs):
        e = rel_err_per_pixel(gc[b], o.c)
        assert np.max(e) <= 1e-4, f"image {b}: max rel err {np.max(e):.3e}"
        assert np.max(np.abs(gmu[b] - o.mu)) <= 1e-3 * max(1.0, np.max(np.abs(o.mu)))  # loose (R18)
        olab, ocnt, _ = oracle.labels(o.c.astype(np.float32), cfg.delta_label)
        assert gcnt[b] == ocnt and np.mean(olab == glab[b]) >= 0.999
    assert len(gst) == cfg.rounds
    if Bn == 1:
        for g, ref in zip(gst, refs[0].stats):
            for key, idx in (("e_tv", 0), ("e_fid", 1), ("primal", 2), ("dual", 3), ("al_residual", 5)):
                assert g[key] == pytest.approx(ref[idx], rel=1e-3, abs=1e-6), key
            assert g["gap"] >= -1e-6


def test_lin_one_step_random_state():
    rng = np.random.default_rng(31)
    H, W, C = 37, 45, 3
    I = rng.random((1, H, W, C), dtype=np.float32)
    h = 1.0 / (W - 1)
    sp = dict(alpha=8.0 / h, beta=1.0, radius=3, kernel=0, eps_x=0.0, eps_c=20.0, dt=0.25, rho=2.5 * h,
              gamma=2.5 * h, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=5, rounds=1, scheme=LIN)
    c0 = np.clip(I + 0.05 * rng.standard_normal(I.shape).astype(np.float32), 0, 1)
    mu0 = (0.3 * rng.standard_normal((1, H, W, 2 * C))).astype(np.float32)
    with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I) as s:
        s.set_field(msa.FIELD_C, c0)
        s.set_field(msa.FIELD_MU, mu0)
        s.step(1)
        gc, gmu = s.get_field(msa.FIELD_C)[0], s.get_field(msa.FIELD_MU)[0]
    o = oracle.State(oracle.Params.from_solver(H, W, C, sp), I[0].astype(np.float64))
    o.c = c0[0].astype(np.float64)
    o.mu = mu0[0].astype(np.float64)
    o.run(1)
    assert np.max(rel_err_per_pixel(gc, o.c)) <= 1e-5
    assert np.max(np.abs(gmu - o.mu)) <= 1e-5


def test_lin_constant_image_fixed_point_bitwise():
    I = np.tile(np.array([0.25, 0.5, 0.875], dtype=np.float32), (1, 33, 40, 1))
    h = 1.0 / 39
    sp = dict(alpha=8.0 / h, beta=1.0, radius=3, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25, rho=2.5 * h,
              gamma=2.5 * h, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=5, rounds=3, scheme=LIN)
    with msa.Solver(msa.Params.from_solver(1, 33, 40, 3, sp), I) as s:
        s.solve()
        assert np.array_equal(s.get_field(msa.FIELD_C), I)
        assert not np.any(s.get_field(msa.FIELD_MU))


HERE = os.path.dirname(os.path.abspath(__file__))


def test_lin_split_bitwise(tmp_path):
    """Rows mode's interior / boundary launches (MSA_K1_SPLIT on one GPU) give identical fields."""
    spec = dict(seed=5, shape=[1, 130, 70, 3], iters=4, random_state=False,
                params=dict(alpha=8.0 * 69, beta=1.0, radius=3, kernel=0, eps_c=20.0, dt=0.25, rho=2.5 / 69,
                            gamma=2.5 / 69, iters_per_round=2, rounds=1, scheme=LIN))
    outs = []
    for split in (False, True):
        env = hook_env()
        env.pop("MSA_K1_SPLIT", None)
        if split:
            env["MSA_K1_SPLIT"] = "1"
        out = str(tmp_path / f"s{int(split)}.npz")
        subprocess.run([sys.executable, os.path.join(HERE, "_run_case.py"), json.dumps(spec), out], check=True,
                       env=env)
        outs.append(np.load(out))
    for k in ("c", "mu"):
        assert np.array_equal(outs[0][k], outs[1][k]), k


@pytest.mark.parametrize("shape,R", [((1, 64, 32, 3), 5), ((1, 130, 97, 3), 5), ((2, 70, 66, 3), 2),
                                     ((1, 37, 29, 3), 3), ((1, 5, 7, 3), 4), ((1, 48, 40, 1), 5),
                                     ((1, 40, 36, 16), 3), ((2, 33, 41, 7), 5), ((1, 9, 70, 12), 2)])
def test_lin_tile_equals_generic_bitwise(shape, R, tmp_path):
    """The tiled kernels of the single-loop scheme (msa_iter_fast.cu LIN for C <= 4, msa_iter_cn.cu
    LIN for C = 5..16) have the generic kernel's per-pixel arithmetic: bitwise-identical fields,
    across a round."""
    B, H, W, C = shape
    h = 1.0 / (W - 1) if W > 1 else 1.0
    spec = dict(seed=H * 100 + W + R, shape=list(shape), iters=3,
                params=dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=0, eps_c=20.0, dt=0.25, rho=2.5 * h,
                            gamma=2.5 * h, iters_per_round=2, rounds=1, scheme=LIN))
    outs = []
    for variant in ("generic", "tile"):
        env = hook_env(MSA_K1=variant)
        env.pop("MSA_FORCE_GENERIC", None)
        out = str(tmp_path / f"{variant}.npz")
        subprocess.run([sys.executable, os.path.join(HERE, "_run_case.py"), json.dumps(spec), out], check=True,
                       env=env)
        outs.append(np.load(out))
    for k in ("c", "mu"):
        assert np.array_equal(outs[0][k], outs[1][k]), (k, float(np.max(np.abs(outs[0][k] - outs[1][k]))))


@pytest.mark.parametrize("name,H,W,B", [("cfg2", 48, 40, None), ("cfg5", 36, 40, 2)])
def test_residual_balancing_matches_oracle(name, H, W, B):
    """msa_solve_until_balanced (residual-balancing rho) against
    oracle.solve_until_balanced (pins RB1-RB3): the same rho in every round's record, dual residuals
    to 1e-3 (R18: loose), the final colour field within the parity gate."""
    cfg, img, sp = config_case(name, H=H, W=W, B=B, rounds=1, iters_per_round=10)
    Bn, Hh, Ww, C = img.shape
    with msa.Solver(msa.Params.from_solver(Bn, Hh, Ww, C, sp), img) as s:
        recs, dres, conv = s.solve_until_balanced(6)
        c = s.get_field(msa.FIELD_C)
    rho_o, dual_o, c_o = [], [], []
    for b in range(Bn):
        st, ro, do = oracle.solve_until_balanced(oracle.Params.from_solver(Hh, Ww, C, sp), img[b], 6)
        rho_o.append([r[6] for r in ro])
        dual_o.append(do)
        c_o.append(st.c)
    if Bn == 1:  # batch records reduce over the images, so the rule sees the batch's residuals
        assert [r["rho"] for r in recs] == pytest.approx(rho_o[0], rel=1e-6)
        assert len(set(r["rho"] for r in recs)) > 1
        np.testing.assert_allclose(dres[1:], np.array(dual_o[0][1:]), rtol=1e-3)
        assert float(rel_err_per_pixel(c[0], c_o[0]).max()) <= 1e-4
    else:
        assert all(np.isfinite(dres[1:])) and np.isnan(dres[0])
        assert len(recs) == 6
