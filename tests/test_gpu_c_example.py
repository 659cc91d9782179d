"""The C ABI from plain C (examples/quantize.c, built by __graft_entry__.build()): init, solve,
labels with palette, free - no Python or torch in the process. Four noisy quadrants must come out
as four clusters whose palette entries are the quadrant colours."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("H,W", [(96, 128), (61, 77)])
def test_c_example_quantizes(H, W):
    import __graft_entry__ as g
    exe = g.build_examples()
    r = subprocess.run([exe, str(H), str(W)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.split()[0] == "ok" and r.stdout.split()[4] == "4", r.stdout


def test_python_quantize_one_call():
    """msa.quantize: the same four-quadrant picture from Python in one call (grey and RGB)."""
    import numpy as np
    msa = pytest.importorskip("paper_2510_16154_b200")
    rng = np.random.default_rng(3)
    H, W = 80, 96
    for C in (1, 3):
        cols = np.array([[0.05], [0.35], [0.65], [0.95]]) if C == 1 else np.array(
            [[0.1, 0.2, 0.8], [0.9, 0.1, 0.1], [0.2, 0.8, 0.3], [0.9, 0.9, 0.2]])
        q = (np.arange(H)[:, None] >= H // 2) * 2 + (np.arange(W)[None, :] >= W // 2)
        img = np.clip(cols[q] + 0.03 * rng.standard_normal((H, W, C)), 0, 1).astype(np.float32)
        c, lab, cnt, pal = msa.quantize(img, delta=0.1, radius=3, iters_per_round=20, rounds=5, max_k=8)
        assert c.shape == (H, W, C) and lab.shape == (H, W)
        assert int(cnt[0]) == 4, (C, cnt, pal[0, :int(cnt[0]), 0])
        assert np.allclose(np.sort(pal[0, :4, 0]), np.sort(cols[:, 0]), atol=0.05)
