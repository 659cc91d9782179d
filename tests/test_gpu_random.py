"""Randomised parity sweep: 150 seeded draws over the whole parameter space the ABI accepts (shape
including 1-pixel axes and ragged tiles, batch, channels 1-16, radius 0-12, both kernels, eps_x
from the default to inside the paper's box, eps_c including 0 and values outside the scaled-form
range, dt, alpha, beta, rho, gamma, kappa, theta, both schemes, K and rounds), each run through the
C ABI and the fp64 oracle on the same image: final colour field to the north_star tolerance (max
per-pixel relative error <= 1e-4) and the per-round rho and primal value. The draws exercise
every K1 variant the dispatcher can pick (tiled C <= 4 with both tile heights, C = 16, generic,
large-support) and both step-1 forms. Draws whose oracle trajectory leaves [-0.5, 1.5] (an
anti-diffusive printed kernel, or a multiplier step gamma > 1.6 rho) are unstable by the method's
own arithmetic and are held to 1e-2 instead (4 of the 150)."""
import numpy as np
import pytest

from _harness import gpu_params, rel_err_per_pixel, run_oracle

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")


def _draw(seed):
    rng = np.random.default_rng(90000 + seed)
    C = int(rng.choice([1, 2, 3, 3, 4, 16, int(rng.integers(5, 16))]))
    H = int(rng.choice([1, int(rng.integers(2, 80))]) if rng.random() < 0.15 else rng.integers(8, 80))
    W = int(rng.integers(1, 90) if rng.random() < 0.15 else rng.integers(8, 90))
    B = int(rng.choice([1, 1, 2]))
    R = int(rng.choice([0, 1, 2, 3, 4, 5, 5, 6, 9, 12]))
    if C > 4 and R > 8:
        R = 5  # large supports are for C <= 4
    scheme = int(rng.random() < 0.3)
    h = 1.0 / (max(W, H) - 1) if max(W, H) > 1 else 1.0
    eps_c = float(rng.choice([0.0, 1e-4, 8.0, 57.0, 300.0, 2500.0]))
    sp = dict(alpha=float(rng.choice([0.0, 1.0, 8.0 / h])) if scheme == 0 else float(rng.choice([1.0, 8.0 / h])),
              beta=float(rng.choice([0.0, 0.5, 1.0])), radius=R, kernel=int(rng.integers(0, 2)),
              eps_x=float(rng.choice([0.0, 0.0, 50.0, 600.0])), eps_c=eps_c, dt=float(rng.choice([0.0, 0.1, 0.25, 0.5])),
              rho=float(rng.uniform(0.5, 4.0) * h), gamma=float(rng.uniform(0.5, 4.0) * h),
              kappa=float(rng.choice([1.0, 1.0, 1.5])) if scheme == 0 else float(rng.choice([1.0, 0.9])),
              tau=0.0, sigma=0.0, theta=float(rng.choice([1.0, 1.0, 0.0, 0.5])),
              iters_per_round=int(rng.integers(1, 8)), rounds=int(rng.integers(1, 4)), scheme=scheme)
    img = rng.random((B, H, W, C), dtype=np.float32)
    if rng.random() < 0.5:  # piecewise-constant structure + noise
        img = np.clip(np.round(img * 3) / 3 + 0.05 * rng.standard_normal(img.shape).astype(np.float32), 0, 1)
    return img.astype(np.float32), sp


@pytest.mark.parametrize("seed", range(150))
def test_random_parameters_match_oracle(seed):
    img, sp = _draw(seed)
    with msa.Solver(gpu_params(img, sp), img) as s:
        st = s.solve()
        gc = s.get_field(msa.FIELD_C)
    refs = run_oracle(img, sp)
    for b, ref in enumerate(refs):
        err = float(np.max(rel_err_per_pixel(gc[b], ref.c)))
        # the printed kernel is repulsive (phi < 0 for r > 1/4): with weak colour decay and weak
        # control it is anti-diffusion, the colours leave [0, 1] and rounding differences grow with
        # the solution; those draws are held to a looser bound (still far below a wrong result)
        tol = 1e-4 if np.all((ref.c > -0.5) & (ref.c < 1.5)) else 1e-2
        assert err <= tol, (seed, sp, img.shape, err)
    for r, o in zip(st, refs[0].stats if img.shape[0] == 1 else []):
        assert r["rho"] == pytest.approx(o[6], rel=1e-12)
        if sp["alpha"] > 0:
            assert r["primal"] == pytest.approx(o[2], rel=1e-3, abs=1e-6)


def _label_field(seed):
    """Fields built to stress stage (ii): few colour levels plus small noise (many segments whose
    means straddle delta and the cell boundaries), random shapes, channel counts and delta."""
    rng = np.random.default_rng(70000 + seed)
    C = int(rng.choice([1, 2, 3, 4, 7, 16]))
    H, W = int(rng.integers(1, 120)), int(rng.integers(1, 120))
    B = int(rng.choice([1, 2]))
    levels = int(rng.integers(2, 6))
    base = np.round(rng.random((B, H, W, C)) * (levels - 1)) / (levels - 1)
    if rng.random() < 0.5:  # blocky regions instead of per-pixel levels
        bh, bw = max(H // int(rng.integers(1, 6)), 1), max(W // int(rng.integers(1, 6)), 1)
        base = np.repeat(np.repeat(base[:, ::bh, ::bw], bh, 1), bw, 2)[:, :H, :W]
    noise = float(rng.choice([0.0, 0.01, 0.03, 0.08]))
    f = np.clip(base + noise * rng.standard_normal(base.shape), 0, 1).astype(np.float32)
    delta = float(rng.choice([0.0, 0.02, 0.05, 0.1, 0.25]))
    return f, delta


@pytest.mark.parametrize("seed", range(60))
def test_random_labels_bitexact(seed):
    """Q(c; delta) on random fields: GPU labels, counts and palettes equal the oracle's bit for bit."""
    f, delta = _label_field(seed)
    B, H, W, C = f.shape
    sp = dict(alpha=1.0, beta=1.0, radius=2, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25, rho=1.0, gamma=1.0,
              kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1, rounds=1)
    with msa.Solver(gpu_params(f, sp), f) as s:  # c = I = f after init
        glab, gcnt, gpal = s.labels(delta, max_k=16)
    import oracle
    for b in range(B):
        olab, ocnt, opal = oracle.labels(f[b], delta, max_k=16)
        assert gcnt[b] == ocnt, (seed, b, gcnt[b], ocnt)
        assert np.array_equal(glab[b], olab), (seed, b)
        k = min(ocnt, 16)
        assert np.array_equal(gpal[b][:k], opal[:k]), (seed, b)
