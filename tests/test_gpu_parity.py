"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
inputs. Tolerances: final colour field max per-pixel relative
error <= 1e-4 (north_star); single iterations <= 1e-5 (fp32 rounding of one step);
labels >= 99.9% equal with an identical count, and bit-exact when both sides label the
same fp32 field."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
import synth
from _harness import config_case, gpu_params, rel_err_per_pixel, run_oracle

pytestmark = pytest.mark.gpu

msa = pytest.importorskip("paper_2510_16154_b200")


def _solver(img, sp, **over):
    return msa.Solver(gpu_params(img, sp, **over), img)


def _rand_state(rng, B, H, W, C, pscale=0.3):
    I = rng.random((B, H, W, C), dtype=np.float32)
    c = np.clip(I + 0.05 * rng.standard_normal((B, H, W, C)).astype(np.float32), 0, 1)
    cb = np.clip(c + 0.02 * rng.standard_normal((B, H, W, C)).astype(np.float32), 0, 1)
    p = (pscale * rng.standard_normal((B, H, W, 2 * C))).astype(np.float32)
    mu = (pscale * rng.standard_normal((B, H, W, 2 * C))).astype(np.float32)
    return I, c, cb, p, mu


def _oracle_state(prm, I, c, cb, p, mu):
    s = oracle.State(prm, I.astype(np.float64))
    s.c[...] = c
    s.cbar[...] = cb
    s.p[...] = p
    s.mu[...] = mu
    return s


@pytest.mark.parametrize("H,W,C,R", [(23, 37, 1, 2), (40, 33, 3, 2), (45, 70, 3, 3), (50, 61, 3, 5),
                                     (19, 29, 16, 3), (17, 9, 2, 4), (1, 40, 3, 2), (33, 1, 3, 3), (1, 1, 3, 2),
                                     (70, 45, 1, 5), (31, 44, 4, 5), (40, 36, 2, 3)])
def test_single_iteration_random_state(H, W, C, R):
    """Steps 1-3 from an arbitrary state: c+, cbar+, p+ element by element."""
    rng = np.random.default_rng(1000 + H * W + C + R)
    I, c, cb, p, mu = _rand_state(rng, 1, H, W, C)
    sp = dict(alpha=3.0 * (W - 1 if W > 1 else 1), beta=1.0, radius=R, kernel=0, eps_x=0.0, eps_c=20.0, dt=0.25,
              rho=0.7, gamma=0.7, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1000, rounds=1)
    with _solver(I, sp) as s:
        for f, a in ((msa.FIELD_C, c), (msa.FIELD_CBAR, cb), (msa.FIELD_P, p), (msa.FIELD_MU, mu)):
            s.set_field(f, a)
        s.step(1)
        gc, gcb, gp = s.get_field(msa.FIELD_C)[0], s.get_field(msa.FIELD_CBAR)[0], s.get_field(msa.FIELD_P)[0]
    o = _oracle_state(oracle.Params.from_solver(H, W, C, sp), I[0], c[0], cb[0], p[0], mu[0])
    o.iteration()
    assert np.max(np.abs(gc - o.c)) <= 1e-5 * max(1.0, np.max(np.abs(o.c)))
    assert np.max(np.abs(gcb - o.cbar)) <= 2e-5 * max(1.0, np.max(np.abs(o.cbar)))
    assert np.max(np.abs(gp - o.p)) <= 1e-5 * max(1.0, np.max(np.abs(o.p)))


@pytest.mark.parametrize("kernel", [0, 1])
def test_single_iteration_printed_kernel(kernel):
    rng = np.random.default_rng(7 + kernel)
    I, c, cb, p, mu = _rand_state(rng, 1, 30, 34, 3)
    sp = dict(alpha=50.0, beta=0.5, radius=3, kernel=kernel, eps_x=500.0, eps_c=8.0, dt=0.5, rho=0.3, gamma=0.3,
              kappa=1.0, tau=0.0, sigma=0.0, theta=0.5, iters_per_round=1000, rounds=1)
    with _solver(I, sp) as s:
        for f, a in ((msa.FIELD_C, c), (msa.FIELD_CBAR, cb), (msa.FIELD_P, p), (msa.FIELD_MU, mu)):
            s.set_field(f, a)
        s.step(1)
        gc = s.get_field(msa.FIELD_C)[0]
    o = _oracle_state(oracle.Params.from_solver(30, 34, 3, sp), I[0], c[0], cb[0], p[0], mu[0])
    o.iteration()
    assert np.max(np.abs(gc - o.c)) <= 1e-5


@pytest.mark.parametrize("C", [1, 3, 16])
def test_round_update_and_stats(C):
    """Steps 4-5: mu+ element by element and the round record (loose, R18)."""
    rng = np.random.default_rng(50 + C)
    H, W = 27, 31
    I, c, cb, p, mu = _rand_state(rng, 1, H, W, C)
    sp = dict(alpha=40.0, beta=1.0, radius=2, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25, rho=0.2, gamma=0.15,
              kappa=1.5, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1, rounds=2)
    with _solver(I, sp) as s:
        for f, a in ((msa.FIELD_C, c), (msa.FIELD_CBAR, cb), (msa.FIELD_P, p), (msa.FIELD_MU, mu)):
            s.set_field(f, a)
        s.step(2)
        gmu = s.get_field(msa.FIELD_MU)[0]
        gc = s.get_field(msa.FIELD_C)[0]
        st = s.stats()
    o = _oracle_state(oracle.Params.from_solver(H, W, C, sp), I[0], c[0], cb[0], p[0], mu[0])
    ost = o.run(2)
    assert np.max(rel_err_per_pixel(gc, o.c)) <= 1e-4
    assert np.max(np.abs(gmu - o.mu)) <= 1e-4 * max(1.0, np.max(np.abs(o.mu)))
    assert len(st) == 2
    for r in range(2):
        g, ref = st[r], ost[r]
        for key, idx in (("e_tv", 0), ("e_fid", 1), ("primal", 2), ("dual", 3), ("al_residual", 5), ("rho", 6)):
            assert g[key] == pytest.approx(ref[idx], rel=1e-3, abs=1e-6), key
        assert g["mean"][:C] == pytest.approx(list(ref[8:8 + C]), rel=1e-5)
        assert g["nonfinite"] == 0


@pytest.mark.parametrize("case", [
    ("cfg1", None, None, None),
    ("cfg2", 96, 80, None),
    ("cfg3", 64, 72, None),
    ("cfg4", 70, 64, None),
    ("cfg5", 40, 48, 2),
])
def test_config_parity(case):
    """Each BASELINE config's recipe and schedule (full iteration count) at a size the oracle
    finishes in seconds: c within 1e-4 per pixel (R17), labels >= 99.9% and equal count."""
    name, H, W, B = case
    cfg, img, sp = config_case(name, H, W, B)
    with _solver(img, sp) as s:
        gst = s.solve()
        gc = s.get_field(msa.FIELD_C)
        glab, gcnt, _ = s.labels(cfg.delta_label)
    refs = run_oracle(img, sp)
    for b, o in enumerate(refs):
        e = rel_err_per_pixel(gc[b], o.c)
        assert np.max(e) <= 1e-4, f"image {b}: max rel err {np.max(e):.3e}"
        olab, ocnt, _ = oracle.labels(o.c.astype(np.float32), cfg.delta_label)
        agree = np.mean(olab == glab[b])
        assert gcnt[b] == ocnt and agree >= 0.999, (gcnt[b], ocnt, agree)
    assert len(gst) == cfg.rounds


@pytest.mark.parametrize("over,C", [
    (dict(radius=8), 16),            # maximum radius and channel count (generic kernel)
    (dict(radius=0), 3),             # no interaction at all (N_R = 1)
    (dict(radius=1), 3),             # R = 1: every neighbour on the ring, phi = 0 (R22)
    (dict(dt=0.0), 3),               # pure primal-dual (P14-P17 regime)
    (dict(alpha=0.0), 2),            # no fidelity: D and gap NaN by definition
    (dict(beta=0.0), 3),             # no TV: p stays 0
    (dict(kappa=1.7, theta=0.0), 3), # penalty growth, no extrapolation
    (dict(eps_x=50.0, radius=4), 3), # small eps_x: ring offsets active -> generic kernel
    (dict(kernel=1), 1),             # printed (repulsive) kernel, grey
    (dict(radius=5), 1),             # grey (the paper's image type) on the tiled kernel, R = 5
    (dict(radius=4), 4),             # RGBA on the tiled kernel (P = 2 tiles)
    # the scaled step-1 form (MsaIterConsts::scaled) holds for e_c = eps_c/2 in [1e-3, 1e3]; outside
    # it the direct form runs (generic kernel): both ends of the range and both sides of it
    (dict(eps_c=0.0), 3),
    (dict(eps_c=1e-4), 3),
    (dict(eps_c=2e-3), 3),
    (dict(eps_c=1999.0), 3),
    (dict(eps_c=2100.0), 3),
])
def test_degenerate_and_extreme_params(over, C):
    rng = np.random.default_rng(len(str(over)) + C)
    H, W = 29, 35
    img = rng.random((1, H, W, C), dtype=np.float32)
    h = 1.0 / (W - 1)
    sp = dict(alpha=8.0 / h, beta=1.0, radius=3, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25, rho=2.5 * h,
              gamma=2.5 * h, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=7, rounds=3)
    sp.update(over)
    with _solver(img, sp) as s:
        st = s.solve()
        gc = s.get_field(msa.FIELD_C)[0]
    ref = run_oracle(img, sp)[0]
    assert np.max(rel_err_per_pixel(gc, ref.c)) <= 1e-4
    if sp["alpha"] == 0:
        assert all(np.isnan(r["dual"]) and np.isnan(r["gap"]) for r in st)
    else:
        for r, o in zip(st, ref.stats):
            assert r["primal"] == pytest.approx(o[2], rel=1e-3, abs=1e-6)
            assert r["rho"] == pytest.approx(o[6], rel=1e-12)
    if sp["beta"] == 0:
        with _solver(img, sp) as s:
            s.solve()
            assert not np.any(s.get_field(msa.FIELD_P))


def test_invalid_shapes_rejected():
    """Empty images and over-size parameters fail with MSA_EINVAL (no partial state)."""
    sp = synth.solver_params(synth.CONFIGS["cfg1"])
    for shape in [(1, 0, 8, 3), (1, 8, 0, 3), (0, 8, 8, 3)]:
        img = np.zeros((max(shape[0], 1), max(shape[1], 1), max(shape[2], 1), 3), np.float32)
        p = gpu_params(img, sp)
        p.batch, p.height, p.width = shape[0], shape[1], shape[2]
        with pytest.raises(msa.MsaError) as e:
            msa.Solver(p, img)
        assert e.value.code == msa.MSA_EINVAL


def test_constant_image_is_fixed_point_bitwise():
    """P9 on the GPU: I constant => c = cbar = I, p = mu = 0 bitwise after every iteration."""
    img = np.full((1, 24, 30, 3), 0.375, dtype=np.float32)
    img[..., 1] = 0.8125
    sp = synth.solver_params(synth.resized(synth.CONFIGS["cfg1"], 24, 30, rounds=3, iters_per_round=7))
    with _solver(img, sp) as s:
        s.solve()
        assert np.array_equal(s.get_field(msa.FIELD_C), img)
        assert np.array_equal(s.get_field(msa.FIELD_CBAR), img)
        assert not np.any(s.get_field(msa.FIELD_P))
        assert not np.any(s.get_field(msa.FIELD_MU))


def test_labels_bitexact_same_field():
    """K4 and the oracle's Q(c; delta) on the same fp32 field give identical labels."""
    cfg, img, sp = config_case("cfg2", 128, 96, rounds=2, iters_per_round=25)
    with _solver(img, sp) as s:
        s.solve()
        gc = s.get_field(msa.FIELD_C)[0]
        glab, gcnt, gpal = s.labels(0.1, max_k=64)
    olab, ocnt, opal = oracle.labels(gc, 0.1, max_k=64)
    assert gcnt[0] == ocnt
    assert np.array_equal(glab[0], olab)
    k = min(ocnt, 64)
    assert np.array_equal(gpal[0][:k], opal[:k])
    # raw noisy input (many segments) too
    with _solver(img, sp) as s:
        glab, gcnt, _ = s.labels(0.05)
    olab, ocnt, _ = oracle.labels(img[0], 0.05)
    assert gcnt[0] == ocnt and np.array_equal(glab[0], olab)


@pytest.mark.parametrize("name,H,W,B,delta", [("cfg3", 384, 320, None, 0.1), ("cfg3", 256, 256, None, 0.02),
                                              ("cfg5", 96, 80, 2, 0.1), ("cfg1", 64, 64, None, 0.0),
                                              ("cfg2", 200, 3, None, 0.1), ("cfg4", 1, 300, None, 0.15)])
def test_labels_bitexact_raw_fields(name, H, W, B, delta):
    """K4 vs the oracle's Q(c; delta) on unsmoothed inputs: many segments, salt-and-pepper outliers,
    C = 16 (no same-cell shortcut), delta = 0, one-pixel-wide images."""
    cfg, img, sp = config_case(name, H, W, B)
    with _solver(img, sp) as s:
        glab, gcnt, gpal = s.labels(delta, max_k=32)
    for b in range(img.shape[0]):
        olab, ocnt, opal = oracle.labels(img[b], delta, max_k=32)
        assert gcnt[b] == ocnt
        assert np.array_equal(glab[b], olab)
        k = min(ocnt, 32)
        assert np.array_equal(gpal[b][:k], opal[:k])


def test_mean_preserved_gpu():
    """P8 on the GPU: the per-channel mean is preserved (fp32 drift only)."""
    cfg, img, sp = config_case("cfg1")
    with _solver(img, sp) as s:
        st = s.solve()
    m0 = img[0].reshape(-1, 3).astype(np.float64).mean(0)
    for r in st:
        assert np.allclose(r["mean"][:3], m0, rtol=0, atol=2e-6)


def test_state_roundtrip_resume_exact():
    cfg, img, sp = config_case("cfg1", rounds=2, iters_per_round=10)
    with _solver(img, sp) as s:
        s.step(13)
        blob = s.get_state()
        s.step(17)
        ref = s.get_field(msa.FIELD_C)
        s.set_state(blob)
        s.step(17)
        assert np.array_equal(s.get_field(msa.FIELD_C), ref)


def test_invalid_params_fail_loudly():
    img = np.zeros((1, 8, 8, 3), np.float32)
    sp = synth.solver_params(synth.CONFIGS["cfg1"])
    with pytest.raises(msa.MsaError) as e:
        msa.Solver(gpu_params(img, dict(sp, rho=-1.0)), img)
    assert e.value.code == msa.MSA_EINVAL
    with pytest.raises(msa.MsaError):
        msa.Solver(gpu_params(img, dict(sp, radius=256)), img)
    with pytest.raises(msa.MsaError):
        msa.Solver(gpu_params(img, dict(sp, scheme=1, kappa=2.0)), img)
