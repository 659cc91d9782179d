"""Row slabs end to end on one GPU: the library's NCCL calls are served by its
in-process loopback transport (MSA_NCCL_LOOPBACK=1, msa_nccl_loopback.cu), and `world` contexts of
one process, one host thread each, run the real row-slab path - partition with ghost rows, the halo
plan executed as grouped send/recv on the comm stream overlapped with the interior K1 launch, the
boundary launches, all-reduced round sums, the labels' all-gathered segment tables and merge.
Checked against one context on the whole image: fields bitwise, labels, counts and palettes
identical, round records to fp64 summation order. Slabs as thin as the ghost width, a ragged split,
R = 5 with the tiled kernel, the C = 16 kernel, the linearised scheme, two images."""
import json
import os
import subprocess
import sys

import pytest
from _harness import hook_env

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(spec, **env_extra):
    env = hook_env(MSA_NCCL_LOOPBACK="1")
    for k in ("MSA_NO_OVERLAP", "MSA_K1", "MSA_FORCE_GENERIC", "MSA_K1_SPLIT", "MSA_LABELS_PARTS"):
        env.pop(k, None)
    env.update(env_extra)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_loopback_case.py"), json.dumps(spec)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def _params(W, R, K=4, rounds=3, **kw):
    h = 1.0 / (W - 1)
    return dict(alpha=8.0 / h, beta=1.0, radius=R, eps_c=57.0, dt=0.25, rho=2.5 * h, gamma=2.5 * h,
                iters_per_round=K, rounds=rounds, **kw)


@pytest.mark.parametrize("shape,R,worlds,extra", [
    ((1, 256, 96, 3), 5, [2, 3], {}),               # tiled K1, interior/boundary split (slabs >= 96 rows)
    ((1, 61, 40, 3), 3, [2, 4], {}),                # ragged slabs, no split, thin slabs
    ((1, 20, 33, 3), 5, [4], {}),                   # slabs exactly the ghost width (5 rows)
    ((2, 200, 64, 3), 4, [2], {"kernel": 1}),       # two images, printed kernel
    ((1, 130, 40, 16), 3, [2], {}),                 # C = 16 kernel
    ((1, 224, 64, 3), 5, [2], {"scheme": 1, "tau": 0.0}),  # single-loop linearised ADMM
    ((1, 96, 48, 3), 12, [2], {}),                  # large support (R > 8)
])
def test_row_slabs_match_one_context(shape, R, worlds, extra):
    spec = dict(seed=sum(shape) + R, shape=list(shape), worlds=worlds, params=_params(shape[2], R, **extra))
    rep = _run(spec)
    for w in worlds:
        assert rep["worlds"][str(w)]["fields"] == "bitwise"


def test_row_slabs_at_the_bench_geometry():
    # the 8-GPU bench geometry of cfg4: 4096^2 RGB, R = 5, eight 512-row slabs (interior / boundary split,
    # the packed halo exchange at full row width), against one context on the whole image
    shape, R = (1, 4096, 4096, 3), 5
    spec = dict(seed=11, shape=list(shape), worlds=[8], params=_params(shape[2], R, K=3, rounds=2))
    rep = _run(spec)
    assert rep["worlds"]["8"]["fields"] == "bitwise" and rep["worlds"]["8"]["labels"] == "identical"


def test_row_slabs_serial_exchange_and_generic_kernel():
    # the exchange on the compute stream before each K1 (MSA_NO_OVERLAP), and the generic kernel
    shape, R = (1, 256, 64, 3), 5
    spec = dict(seed=5, shape=list(shape), worlds=[2], params=_params(shape[2], R))
    assert _run(spec, MSA_NO_OVERLAP="1")["worlds"]["2"]["fields"] == "bitwise"
    assert _run(spec, MSA_K1="generic")["worlds"]["2"]["fields"] == "bitwise"


def test_batch_shards_match_one_context():
    # shard = batch (cfg 5's mode): no data-path collective; every rank's images equal the
    # one-context run bit for bit, uneven splits included (5 images over 2 and 3 ranks)
    shape, R = (5, 40, 36, 16), 3
    spec = dict(seed=11, shape=list(shape), worlds=[2, 3], shard="batch", params=_params(shape[2], R))
    rep = _run(spec)
    assert rep["worlds"]["3"]["images"] in ([2, 2, 1], [2, 1, 2], [1, 2, 2])


@pytest.mark.parametrize("seed", range(12))
def test_row_slabs_random(seed):
    """Random slab worlds: shape, channels, radius (up to the slab height), world 2-4, scheme."""
    import numpy as np
    rng = np.random.default_rng(5000 + seed)
    world = int(rng.integers(2, 5))
    R = int(rng.choice([1, 2, 3, 4, 5, 9]))
    C = int(rng.choice([1, 2, 3, 4, 16]))
    if C == 16 and R > 8:
        R = 4
    H = int(rng.integers(max(R, 1) * world, 140))
    W = int(rng.integers(8, 70))
    B = int(rng.choice([1, 2]))
    scheme = int(rng.random() < 0.3)
    extra = {"scheme": scheme, "tau": 0.0} if scheme else {"kernel": int(rng.integers(0, 2))}
    spec = dict(seed=seed, shape=[B, H, W, C], worlds=[world], params=_params(W, R, **extra))
    assert _run(spec)["worlds"][str(world)]["fields"] == "bitwise"
