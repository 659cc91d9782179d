"""Reading R17's decision margin of the quantisation rule (msa_label_margin): per image, the distance of
the closest stage-(i) comparison | ||c_a - c_b||_inf - delta | from flipping, computed on the device in
fp32 exactly as stage (i) compares. Checked bitwise against the same fp32 arithmetic written out with
numpy on the GPU's own field, single image, batch, and a row-slab world through the testing build's
in-process transport (the margin is all-reduced over slabs and must equal the one-context value)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import synth
from _harness import gpu_params, hook_env

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")
HERE = os.path.dirname(os.path.abspath(__file__))


def margin_np(c: np.ndarray, delta: float) -> float:
    c = c.astype(np.float32)
    d = np.float32(delta)
    dr = np.max(np.abs(c[:, 1:] - c[:, :-1]), axis=-1)
    du = np.max(np.abs(c[1:, :] - c[:-1, :]), axis=-1)
    m = [np.min(np.abs(x - d)) for x in (dr, du) if x.size]
    return float(min(m)) if m else float("inf")


@pytest.mark.parametrize("name,H,W,B", [("cfg1", 64, 64, None), ("cfg2", 96, 80, None), ("cfg5", 40, 36, 3)])
def test_margin_matches_fp32_definition(name, H, W, B):
    cfg = synth.resized(synth.CONFIGS[name], H, W, batch=B, rounds=2, iters_per_round=10)
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    with msa.Solver(gpu_params(img, sp), img) as s:
        s.solve()
        c = s.get_field(msa.FIELD_C)
        m = s.label_margin(cfg.delta_label)
    assert m.shape == (img.shape[0],)
    for b in range(img.shape[0]):
        assert m[b] == np.float32(margin_np(c[b], cfg.delta_label)), (b, m[b])


def test_margin_over_row_slabs_equals_one_context(tmp_path):
    script = r"""
import json, sys, threading, numpy as np
sys.path.insert(0, %r)
import paper_2510_16154_b200 as msa
spec = json.loads(sys.argv[1])
rng = np.random.default_rng(5)
B, H, W, C = 1, 90, 70, 3
I = np.clip(np.repeat(np.repeat(rng.random((1, 6, 5, C)), 15, 1), 14, 2) + 0.03 * rng.standard_normal((B, H, W, C)), 0, 1).astype(np.float32)
base = dict(batch=B, height=H, width=W, channels=C, alpha=8 * 69, beta=1.0, radius=3, eps_c=57.0, dt=0.25, rho=2.5 / 69, gamma=2.5 / 69, iters_per_round=4, rounds=2)
with msa.Solver(msa.Params(**base), I) as s:
    s.solve(); ref = float(s.label_margin(0.1)[0])
nid = msa.nccl_unique_id(); out = [None] * 3
def run(r):
    with msa.Solver(msa.Params(**base, shard=msa.SHARD_ROWS, rank=r, world=3, nccl_id=nid), I) as s:
        s.solve(); out[r] = float(s.label_margin(0.1)[0])
ts = [threading.Thread(target=run, args=(r,)) for r in range(3)]
[t.start() for t in ts]; [t.join() for t in ts]
print(json.dumps({"ref": ref, "slabs": out}))
""" % os.path.dirname(HERE)
    r = subprocess.run([sys.executable, "-c", script, "{}"], env=hook_env(MSA_NCCL_LOOPBACK="1"), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(v == res["ref"] for v in res["slabs"]), res
