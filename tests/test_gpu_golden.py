"""Full-size, full-length parity against the oracle on BASELINE.json's five configs (and the cfg4
recipe at 1024^2, which runs the bench's P = 4 tiles through all 10 rounds).

The references in tests/golden/full_<case>.npz were written by tools/make_fullsize_golden.py, which
calls only oracle/ (fp64, Alg. 2 PAPER.md:448-461 in the fused reading R1) and synth/: sampled
pixels of the final colour field (corners, border points, 4096 uniform), the round records, the
oracle's full label map Q(c; delta) (R16) and its cluster counts, and a hash of the input image.

The GPU runs exactly the bench path: msa_solve (graph replay, the default kernels and launch
configuration) from the same generator image at full size. Gates (north_star, R17, R18):
  * c: max per-pixel relative error e(n) <= 1e-4 on every sampled pixel;
  * labels: >= 99.9 % of pixels carry the same canonical label, and the cluster count is equal;
  * round records (loose, duals are not unique - R18): E_TV, E_fid, P and the AL residual within
    1e-3 relative.
"""
import hashlib
import os

import numpy as np
import pytest

import synth
from _harness import gpu_params, rel_err_per_pixel

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg4_1024", "cfg5"]


def _config(name):
    if name == "cfg4_1024":
        return synth.resized(synth.CONFIGS["cfg4"], 1024, 1024)
    return synth.CONFIGS[name]


@pytest.mark.parametrize("name", CASES)
def test_fullsize_full_length_parity(name):
    path = os.path.join(GOLDEN, f"full_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tools/make_fullsize_golden.py {name})")
    ref = np.load(path)
    cfg = _config(name)
    img = synth.generate(cfg.recipe)
    assert hashlib.sha256(img.tobytes()).digest() == ref["input_sha256"].tobytes(), "generator drifted"
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    assert int(ref["iters"]) == cfg.iters
    with msa.Solver(gpu_params(img, sp), img) as s:
        stats = s.solve()
        c = s.get_field(msa.FIELD_C)
        lab, cnt, _ = s.labels(cfg.delta_label)
        margin = s.label_margin(cfg.delta_label)
    idx = ref["idx"]
    worst = 0.0
    for b in range(B):
        e = rel_err_per_pixel(c[b][idx[:, 0], idx[:, 1]], ref["c"][b])
        worst = max(worst, float(e.max()))
        assert e.max() <= 1e-4, (name, b, float(e.max()))
        assert cnt[b] == int(ref["count"][b]), (name, b, int(cnt[b]), int(ref["count"][b]))
        if b < ref["labels"].shape[0]:  # full label map stored (cfg5: the first 4 of 32 images)
            agree = float(np.mean(lab[b] == ref["labels"][b].astype(np.int32)))
            assert agree >= 0.999, (name, b, agree)
        if "labels_sampled" in ref:  # every image: the sampled pixels' canonical labels
            agree_s = float(np.mean(lab[b][idx[:, 0], idx[:, 1]] == ref["labels_sampled"][b].astype(np.int32)))
            assert agree_s >= 0.999, (name, b, agree_s)
    # records are reduced over the context's images: sums of E_TV, E_fid, P; the AL residual is a norm
    for r, rec in enumerate(stats[:cfg.rounds]):
        o = ref["stats"][:, r, :]
        want = {"e_tv": o[:, 0].sum(), "e_fid": o[:, 1].sum(), "primal": o[:, 2].sum(),
                "al_residual": float(np.sqrt((o[:, 5] ** 2).sum()))}
        for key, v in want.items():
            assert abs(rec[key] - v) <= 1e-3 * max(abs(v), 1e-12), (name, r, key, rec[key], v)
    # R17: report the decision margins (oracle field / GPU field); a label that differs between the two
    # can only come from a comparison closer to delta than the fields' difference
    print(f"{name}: max rel err {worst:.2e}, counts {list(map(int, cnt[:B]))}, stage-(i) margin "
          f"oracle {float(np.min(ref['margin'])):.3g} gpu {float(np.min(margin)):.3g}")
