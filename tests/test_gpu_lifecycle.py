"""Context lifecycle on the device: repeated msa_init / solve (captured and replayed CUDA graphs) /
labels / DAL / msa_free leave no device memory behind, with the library's own workspace and with a
caller (torch) workspace, and two contexts used alternately on their own streams give the same
results as one at a time."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
msa = pytest.importorskip("paper_2510_16154_b200")
torch = pytest.importorskip("torch")


def _params(H=48, W=40, C=3, R=3, **kw):
    h = 1.0 / (W - 1)
    base = dict(batch=1, height=H, width=W, channels=C, alpha=8.0 / h, beta=1.0, radius=R, eps_c=57.0, dt=0.25,
                rho=2.5 * h, gamma=2.5 * h, iters_per_round=4, rounds=3)
    base.update(kw)
    return msa.Params(**base)


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return torch.cuda.mem_get_info()[0]


@pytest.mark.parametrize("torch_ws", [True, False])
def test_no_device_memory_left_behind(torch_ws):
    rng = np.random.default_rng(0)
    I = rng.random((1, 48, 40, 3), dtype=np.float32)
    p, pl = _params(), _params(R=12)
    with msa.Solver(p, I, torch_workspace=torch_ws) as s:  # first use: lazy module loads, caches
        s.solve(); s.solve(); s.labels(0.1, 8)
    base = _free()
    for it in range(12):
        with msa.Solver(p, I, torch_workspace=torch_ws) as s:
            s.solve()
            s.solve()                      # graph replay
            s.labels(0.1, 8)
        with msa.Solver(pl, I, torch_workspace=torch_ws) as s:
            eps = np.stack([np.full(4, 40.0), np.full(4, 57.0)], axis=1)
            s.dal_gradient(msa.DalParams(steps=4), eps)
    leaked = base - _free()
    assert leaked <= 8 << 20, leaked


def test_two_contexts_interleaved_match_sequential():
    rng = np.random.default_rng(1)
    I1 = rng.random((1, 48, 40, 3), dtype=np.float32)
    I2 = rng.random((1, 48, 40, 3), dtype=np.float32)
    p = _params()
    ref = []
    for I in (I1, I2):
        with msa.Solver(p, I) as s:
            s.solve(); s.solve()
            ref.append(s.get_field(msa.FIELD_C))
    with msa.Solver(p, I1) as a, msa.Solver(p, I2) as b:
        for _ in range(2):
            a.solve()
            b.solve()
        got = [a.get_field(msa.FIELD_C), b.get_field(msa.FIELD_C)]
    for r, g in zip(ref, got):
        assert np.array_equal(r, g)
