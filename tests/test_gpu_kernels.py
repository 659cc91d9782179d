"""K1 variants against the generic kernel (msa_kernels.cu), over tile-aligned, ragged and tiny
shapes, every specialised radius, both kernel forms, and across a multiplier round:
  * every variant evaluates step 1 in the scaled form (msa_common.cuh MsaIterConsts::scaled); the
    direct form (MSA_NO_SCALED=1, generic kernel) agrees with it to fp32 rounding;
  * the tiled kernel (msa_iter_fast.cu) has the generic kernel's per-pixel arithmetic and term order:
    bitwise-identical fields;
  * the pair-symmetric sweep kernel (msa_iter_sweep.cu) evaluates each pair weight once and sums the
    terms in another (fixed) order: p+ of one iteration is bitwise equal (it does not depend on the
    agent sums), c and cbar agree to fp32 rounding, and its results are bitwise independent of the
    segment length (MSA_SWEEP_SEG) and reproducible run to run."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
from _harness import hook_env

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(spec, variant: str, tmp_path, seg: int = 0, split: bool = False, direct: bool = False, rows_per_thread: int = 0):
    out = str(tmp_path / f"{variant}_{seg}_{int(split)}_{int(direct)}_{rows_per_thread}.npz")
    env = hook_env()
    env.pop("MSA_K1_P", None)
    if rows_per_thread:
        env["MSA_K1_P"] = str(rows_per_thread)
    env.pop("MSA_FORCE_GENERIC", None)
    env.pop("MSA_NO_SCALED", None)
    if direct:
        env["MSA_NO_SCALED"] = "1"
    env["MSA_K1"] = variant
    if split:
        env["MSA_K1_SPLIT"] = "1"
    else:
        env.pop("MSA_K1_SPLIT", None)
    if seg:
        env["MSA_SWEEP_SEG"] = str(seg)
    else:
        env.pop("MSA_SWEEP_SEG", None)
    subprocess.run([sys.executable, os.path.join(HERE, "_run_case.py"), json.dumps(spec), out], check=True, env=env)
    return np.load(out)


CASES = [
    ((1, 64, 32, 3), 5, 0), ((1, 130, 97, 3), 5, 0), ((1, 37, 29, 3), 3, 0), ((2, 70, 66, 3), 2, 1),
    ((1, 5, 7, 3), 4, 0), ((1, 1, 50, 3), 2, 0), ((1, 200, 3, 3), 3, 0), ((1, 256, 256, 3), 5, 1),
]
# many-channel tiled kernel (msa_iter_cn.cu, C = 16): same contract, bitwise equal to the generic one
CN_CASES = [((2, 40, 36, 16), 3, 0), ((1, 33, 70, 16), 4, 1), ((1, 9, 5, 16), 2, 0), ((1, 64, 64, 16), 1, 0),
            ((1, 40, 36, 5), 3, 0), ((2, 33, 41, 8), 4, 1), ((1, 50, 64, 12), 2, 0), ((1, 17, 90, 7), 3, 0),
            ((1, 45, 70, 16), 5, 0), ((1, 37, 29, 6), 5, 1),
            # more tiles (10 x 26 x 2 = 520) than persistent CTAs (2 x 148): each CTA walks several tiles
            ((2, 203, 290, 16), 3, 0)]
# the tiled kernel for grey (the paper's images), two-channel and RGBA fields (C = 1, 2, 4)
C_CASES = [((1, 64, 32, 1), 5, 0), ((2, 70, 45, 1), 3, 1), ((1, 37, 29, 2), 4, 0), ((1, 100, 66, 2), 5, 0),
           ((1, 48, 40, 4), 5, 0), ((2, 33, 70, 4), 2, 1), ((1, 1, 50, 1), 2, 0)]


def _spec(shape, R, ker, iters=3):
    B, H, W, C = shape
    h = 1.0 / (W - 1) if W > 1 else 1.0
    return dict(seed=H * 1000 + W + R, shape=list(shape), iters=iters,
                params=dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=ker, eps_c=20.0, dt=0.25, rho=2.5 * h,
                            gamma=2.5 * h, iters_per_round=2, rounds=1))


@pytest.mark.parametrize("shape,R,ker", CASES + CN_CASES + C_CASES)
def test_tile_equals_generic_bitwise(shape, R, ker, tmp_path):
    spec = _spec(shape, R, ker)
    a = _run(spec, "generic", tmp_path)
    b = _run(spec, "tile", tmp_path)
    for k in ("c", "cbar", "p", "mu"):
        assert np.array_equal(a[k], b[k]), (k, float(np.max(np.abs(a[k] - b[k]))))


# The bench configuration (cfg4, 4096^2) runs the tiled kernel with P = 4 rows per thread (32 x 32
# tiles), which the launcher picks only when the image has at least 2 x 148 tiles; small test images
# pick P = 2. MSA_K1_P=4 forces the bench's P = 4 tiles on small shapes: bitwise equal to the generic
# kernel across two multiplier rounds (5 iterations, K = 2), ragged and tile-aligned.
P4_CASES = [((1, 100, 70, 3), 5, 0), ((1, 64, 64, 3), 5, 1), ((2, 45, 61, 3), 3, 0), ((1, 130, 33, 3), 4, 0),
            ((1, 70, 97, 1), 5, 0), ((1, 41, 40, 2), 2, 1), ((1, 7, 300, 3), 5, 0)]


@pytest.mark.parametrize("shape,R,ker", P4_CASES)
def test_tile_p4_equals_generic_bitwise_across_rounds(shape, R, ker, tmp_path):
    spec = _spec(shape, R, ker, iters=5)
    a = _run(spec, "generic", tmp_path)
    b = _run(spec, "tile", tmp_path, rows_per_thread=4)
    for k in ("c", "cbar", "p", "mu"):
        assert np.array_equal(a[k], b[k]), (k, float(np.max(np.abs(a[k] - b[k]))))


# the sweep kernel is opt-in (MSA_K1=sweep): a representative subset - every radius, both kernels,
# batch, ragged and thin shapes
SWEEP_CASES = [((1, 64, 32, 3), 5, 0), ((1, 37, 29, 3), 3, 0), ((2, 70, 66, 3), 2, 1), ((1, 5, 7, 3), 4, 0),
               ((1, 97, 131, 3), 5, 0), ((3, 45, 61, 3), 3, 1), ((1, 4, 200, 3), 2, 0)]


@pytest.mark.parametrize("shape,R,ker", SWEEP_CASES)
def test_sweep_matches_generic(shape, R, ker, tmp_path):
    # one iteration: p+ does not depend on the agent sums -> bitwise; c, cbar to fp32 rounding
    spec1 = _spec(shape, R, ker, iters=1)
    a = _run(spec1, "generic", tmp_path)
    b = _run(spec1, "sweep", tmp_path)
    assert np.array_equal(a["p"], b["p"])
    assert np.array_equal(a["mu"], b["mu"])
    for k in ("c", "cbar"):
        err = np.max(np.abs(a[k] - b[k]))
        assert err <= 2e-6, (k, float(err))
    # three iterations across a multiplier round
    spec = _spec(shape, R, ker)
    a = _run(spec, "generic", tmp_path)
    b = _run(spec, "sweep", tmp_path)
    for k in ("c", "cbar", "p", "mu"):
        scale = max(1.0, float(np.max(np.abs(a[k]))))
        err = np.max(np.abs(a[k] - b[k])) / scale
        assert err <= 2e-5, (k, float(err))


@pytest.mark.parametrize("shape,R", [((1, 130, 97, 3), 5), ((2, 70, 66, 3), 3), ((1, 37, 29, 3), 2)])
def test_sweep_segment_invariant_and_reproducible(shape, R, tmp_path):
    spec = _spec(shape, R, 0)
    ref = _run(spec, "sweep", tmp_path)
    again = _run(spec, "sweep", tmp_path, seg=0)
    for seg in (1, 3, 7):
        other = _run(spec, "sweep", tmp_path, seg=seg)
        for k in ("c", "cbar", "p", "mu"):
            assert np.array_equal(ref[k], other[k]), (seg, k)
    for k in ("c", "cbar", "p", "mu"):
        assert np.array_equal(ref[k], again[k]), k


# Rows mode runs K1 as an interior launch (overlapped with the NCCL halo exchange) plus two
# boundary launches. MSA_K1_SPLIT=1 runs that split on one GPU: every pixel is
# computed by the same kernel with the same arithmetic, so the fields must be bitwise equal.
@pytest.mark.parametrize("shape,R,variant", [((1, 130, 97, 3), 5, "tile"), ((1, 200, 64, 3), 3, "generic"),
                                             ((2, 100, 36, 16), 3, "tile"), ((1, 96, 40, 3), 2, "tile")])
def test_k1_interior_boundary_split_bitwise(shape, R, variant, tmp_path):
    spec = _spec(shape, R, 0, iters=3)
    a = _run(spec, variant, tmp_path)
    b = _run(spec, variant, tmp_path, split=True)
    for k in ("c", "cbar", "p", "mu"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("shape,R,ker", [((1, 64, 32, 3), 5, 0), ((1, 37, 29, 3), 3, 1), ((2, 40, 36, 16), 3, 0),
                                        ((1, 48, 40, 3), 12, 0), ((1, 30, 33, 1), 2, 0)])
def test_scaled_form_matches_direct_form(shape, R, ker, tmp_path):
    # t = e_c t', phi(t) = e_c^4 phi-part(t'): the same weights up to fp32 rounding of the
    # rescaled offset constants and of e_c^4 dt / N_R
    spec = _spec(shape, R, ker)
    a = _run(spec, "tile", tmp_path)
    b = _run(spec, "tile", tmp_path, direct=True)
    for k in ("c", "cbar", "p", "mu"):
        scale = max(1.0, float(np.max(np.abs(b[k]))))
        err = float(np.max(np.abs(a[k] - b[k]))) / scale
        assert err <= 2e-5, (k, err)
