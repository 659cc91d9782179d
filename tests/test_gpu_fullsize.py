"""Parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times (same kernels,
tiles and grid). The oracle cannot follow 1000 iterations at 4096², so the checks are:
  * sampled pixels after a few iterations, each computed by the oracle on a crop that carries the
    full image's spacing and extends n_iters x reach beyond the sample (exact by locality: see
    tests/test_oracle_pins.py::test_crop_locality_exact), including crops touching image borders;
  * properties that hold at any size after the full solve: per-channel mean preserved, finite
    state, no diverged round, gap/residual finite;
  * labels of the GPU's final field equal the oracle's Q(c; delta) on the same fp32 field, bitwise.
"""
import numpy as np
import pytest

import oracle
import synth
from _harness import gpu_params

pytestmark = pytest.mark.gpu

msa = pytest.importorskip("paper_2510_16154_b200")

N_ITERS = 2


def _crop_check(img_b, sp, gpu_c, H, W, C, boxes, n_iters):
    reach = sp["radius"] + 2
    m = n_iters * reach
    for (j0, j1, i0, i1) in boxes:
        cj0, cj1, ci0, ci1 = max(0, j0 - m), min(H, j1 + m), max(0, i0 - m), min(W, i1 + m)
        prm = oracle.Params.from_solver(cj1 - cj0, ci1 - ci0, C, sp)
        prm.hx, prm.hy = 1.0 / (W - 1), 1.0 / (H - 1)
        prm.iters_per_round = 10 ** 6  # no round inside the sampled iterations
        st = oracle.State(prm, img_b[cj0:cj1, ci0:ci1].astype(np.float64))
        st.run(n_iters)
        ref = st.c[j0 - cj0:j1 - cj0, i0 - ci0:i1 - ci0]
        got = gpu_c[j0:j1, i0:i1].astype(np.float64)
        err = np.max(np.abs(got - ref) / np.maximum(np.max(np.abs(ref), -1, keepdims=True), 1e-3))
        assert err <= 1e-5, (j0, i0, err)


def _boxes(H, W, rng, n=4, size=24):
    bx = [(0, size, 0, size), (H - size, H, W - size, W)]  # corners (image borders)
    for _ in range(n):
        j = int(rng.integers(0, H - size)); i = int(rng.integers(0, W - size))
        bx.append((j, j + size, i, i + size))
    return bx


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_fullsize_sampled_iterations(name):
    cfg = synth.CONFIGS[name]
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    rng = np.random.default_rng(hash(name) % 2 ** 32)
    with msa.Solver(gpu_params(img, sp), img) as s:
        s.step(N_ITERS)
        c = s.get_field(msa.FIELD_C)
    for b in ([0, B - 1] if B > 1 else [0]):
        _crop_check(img[b], sp, c[b], H, W, C, _boxes(H, W, rng), N_ITERS)


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_fullsize_solve_properties_and_labels(name):
    cfg = synth.CONFIGS[name]
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    with msa.Solver(gpu_params(img, sp), img) as s:
        stats = s.solve()
        assert len(stats) == cfg.rounds
        c0 = s.get_field(msa.FIELD_C)[0]
        lab, cnt, _ = s.labels(cfg.delta_label)
    m_in = img.reshape(B, -1, C).astype(np.float64).mean(1).mean(0)
    for r in stats:
        assert r["nonfinite"] == 0
        assert np.isfinite(r["gap"]) and np.isfinite(r["al_residual"])
        assert np.allclose(r["mean"][:C], m_in, rtol=0, atol=5e-5)
    assert np.all(np.isfinite(c0))
    olab, ocnt, _ = oracle.labels(c0, cfg.delta_label)
    assert cnt[0] == ocnt
    assert np.array_equal(lab[0], olab)
