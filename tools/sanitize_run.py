"""Small workloads over every kernel family of the product library, for compute-sanitizer (SURVEY §5:
memcheck, racecheck, synccheck, initcheck on small configs). Host (numpy) inputs, a library-allocated
workspace and the library's own stream, so the only kernels in the process are libmsa.so's.
usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [case ...]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_16154_b200 as msa  # noqa: E402


def image(B, H, W, C, seed):
    rng = np.random.default_rng(seed)
    blocks = np.repeat(np.repeat(rng.random((B, 4, 4, C)), (H + 3) // 4, 1), (W + 3) // 4, 2)[:, :H, :W]
    return np.clip(blocks + 0.05 * rng.standard_normal((B, H, W, C)), 0, 1).astype(np.float32)


def params(B, H, W, C, R, **kw):
    h = 1.0 / (max(H, W) - 1)
    d = dict(batch=B, height=H, width=W, channels=C, alpha=8.0 * h, beta=1.0, radius=R, eps_c=57.0, dt=0.25,
             rho=2.5 * h, gamma=2.5 * h, iters_per_round=2, rounds=2)
    d.update(kw)
    return msa.Params(**d)


def run_solver(p, img, labels=True):
    with msa.Solver(p, img, stream=0, torch_workspace=False) as s:
        s.solve()
        if labels:
            s.labels(0.1, max_k=64)
            s.label_margin(0.1)
        s.get_field(msa.FIELD_C)
        blob = s.get_state()
        s.set_state(blob)
        s.step(1)
        s.sync()


CASES = {
    # tiled K1 (C = 3, 32 x 16 tiles on a small image), round, reduce, record, labels, margin, state
    "rgb_small": lambda: run_solver(params(1, 72, 80, 3, 2), image(1, 72, 80, 3, 0)),
    # tiled K1 with 32 x 32 tiles (P = 4: at least 2 x 148 tiles), masked border tiles, R = 5
    "rgb_p4": lambda: run_solver(params(1, 576, 544, 3, 5, iters_per_round=1, rounds=1), image(1, 576, 544, 3, 1),
                                 labels=False),
    # grey and two-channel tiled kernels
    "grey": lambda: run_solver(params(1, 40, 52, 1, 3), image(1, 40, 52, 1, 2)),
    "two": lambda: run_solver(params(2, 33, 41, 2, 4), image(2, 33, 41, 2, 3)),
    # many-channel K1 (C = 16, batch of two)
    "c16": lambda: run_solver(params(2, 24, 40, 16, 3), image(2, 24, 40, 16, 4)),
    # large-support step 1 (R >= 6)
    "large": lambda: run_solver(params(1, 48, 44, 3, 9), image(1, 48, 44, 3, 5)),
    # generic kernel (C = 5..16 beyond R = 5) and the single-loop linearised scheme
    "generic": lambda: run_solver(params(1, 20, 24, 6, 7), image(1, 20, 24, 6, 6)),
    "lin": lambda: run_solver(params(1, 40, 64, 3, 3, scheme=msa.SCHEME_LINEARISED_ADMM, tau=0.0),
                              image(1, 40, 64, 3, 7)),
    "lin_c16": lambda: run_solver(params(1, 24, 40, 16, 2, scheme=msa.SCHEME_LINEARISED_ADMM, tau=0.0),
                                  image(1, 24, 40, 16, 8)),
}


def dal():
    # NEXT-1: forward sweep, discrete adjoint, eps reductions, Armijo loop (Algorithm 1)
    I = image(1, 16, 16, 3, 9)
    p = params(1, 16, 16, 3, 15, rho=0.5, gamma=0.5, iters_per_round=1, rounds=1)
    eps = np.stack([np.full(6, 100.0), np.full(6, 60.0)], axis=1)
    with msa.Solver(p, I, stream=0, torch_workspace=False) as s:
        s.dal_gradient(msa.DalParams(steps=6), eps)
        s.dal(msa.DalParams(steps=6, iters=2), eps)


CASES["dal"] = dal

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("ok", n, flush=True)
