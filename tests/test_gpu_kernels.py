"""The specialised K1 (msa_iter_fast.cu) against the generic kernel: bitwise-identical fields
(same per-pixel arithmetic and term order), over tile-aligned, ragged and tiny shapes, every
specialised radius, both kernel forms, and across a multiplier round."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(spec, generic: bool, tmp_path):
    out = str(tmp_path / ("gen.npz" if generic else "fast.npz"))
    env = dict(os.environ)
    if generic:
        env["MSA_FORCE_GENERIC"] = "1"
    else:
        env.pop("MSA_FORCE_GENERIC", None)
    subprocess.run([sys.executable, os.path.join(HERE, "_run_case.py"), json.dumps(spec), out], check=True, env=env)
    return np.load(out)


CASES = [
    ((1, 64, 32, 3), 5, 0), ((1, 130, 97, 3), 5, 0), ((1, 37, 29, 3), 3, 0), ((2, 70, 66, 3), 2, 1),
    ((1, 5, 7, 3), 4, 0), ((1, 1, 50, 3), 2, 0), ((1, 200, 3, 3), 3, 0), ((1, 256, 256, 3), 5, 1),
]


@pytest.mark.parametrize("shape,R,ker", CASES)
def test_fast_equals_generic_bitwise(shape, R, ker, tmp_path):
    B, H, W, C = shape
    h = 1.0 / (W - 1) if W > 1 else 1.0
    spec = dict(seed=H * 1000 + W + R, shape=list(shape), iters=3,
                params=dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=ker, eps_c=20.0, dt=0.25, rho=2.5 * h,
                            gamma=2.5 * h, iters_per_round=2, rounds=1))
    a = _run(spec, True, tmp_path)
    b = _run(spec, False, tmp_path)
    for k in ("c", "cbar", "p", "mu"):
        assert np.array_equal(a[k], b[k]), (k, float(np.max(np.abs(a[k] - b[k]))))
