"""Row-slab mode over REAL NCCL (two processes, one GPU each; skipped when fewer than 2 GPUs are
visible - the development pool has one). The slabs must reassemble the one-GPU fields bitwise
(P19), labels and counts must be identical, and the per-rank halo timing must be
reported. The R = 40 case has slabs of 100+ rows and R > 32: the interior launch must then start
R + 1 rows from the slab edges (a fixed 32-row split would read ghost rows the
exchange is still writing)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from _loopback_case import FIELDS, image  # noqa: E402


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


CASES = [
    dict(seed=1, shape=[1, 256, 128, 3], params=dict(alpha=8 * 127, beta=1.0, radius=5, eps_c=57.0, dt=0.25,
                                                      rho=2.5 / 127, gamma=2.5 / 127, iters_per_round=5, rounds=2)),
    # C = 5 at R = 40 runs the generic K1 (which splits; the large-support kernels do not): slabs of
    # 200 rows, interior rows [64, 128)
    dict(seed=2, shape=[1, 400, 64, 5], params=dict(alpha=8 * 63, beta=1.0, radius=40, eps_c=57.0, dt=0.25,
                                                     rho=2.5 / 63, gamma=2.5 / 63, iters_per_round=3, rounds=2)),
    dict(seed=3, shape=[2, 130, 64, 16], params=dict(alpha=8 * 63, beta=1.0, radius=3, eps_c=57.0, dt=0.25,
                                                      rho=2.5 / 63, gamma=2.5 / 63, iters_per_round=4, rounds=2)),
]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs (real NCCL row slabs)")
@pytest.mark.parametrize("spec", CASES, ids=["rgb_R5", "R40_split_margin", "C16_batch2"])
def test_row_slabs_over_nccl_bitwise_equal_one_gpu(spec, tmp_path):
    world = 2
    out = str(tmp_path / "rank")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + spec["seed"]),
           os.path.join(HERE, "_nccl_rank.py"), json.dumps(spec), out]
    subprocess.run(cmd, check=True, timeout=600)
    B, H, W, C = spec["shape"]
    I = image(np.random.default_rng(spec["seed"]), B, H, W, C)
    p = msa.Params(batch=B, height=H, width=W, channels=C, **spec["params"])
    with msa.Solver(p, I) as s:
        s.solve()
        s.solve()
        s.step(p.iters_per_round)
        ref = {k: s.get_field(w) for k, w in FIELDS}
        lab, cnt, pal = s.labels(0.1, 64)
    for r in range(world):
        o = np.load(f"{out}_{r}.npz")
        sl = slice(int(o["row0"]), int(o["row0"]) + int(o["nrows"]))
        for k, _ in FIELDS:
            assert np.array_equal(o[k], ref[k][:, sl]), (r, k)
        assert np.array_equal(o["lab"], lab[:, sl]) and np.array_equal(o["cnt"], cnt)
        assert int(o["halo_exchanges"]) >= p.iters_per_round and float(o["halo_ms"]) > 0.0
