"""Times the DAL building blocks (NEXT-1) at a paper-like size: one cost evaluation (forward sweep
of M Euler steps), one gradient (forward sweep with trajectory + backward sweep), and a short
Algorithm-1 run. usage: python tools/time_dal.py H W R M [iters]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402

H, W, R, M = (int(a) for a in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 2
rng = np.random.default_rng(0)
C = 3
blocks = np.repeat(np.repeat(rng.random((8, 8, C)), H // 8, 0), W // 8, 1)
I = np.clip(blocks + 0.05 * rng.standard_normal((H, W, C)), 0, 1).astype(np.float32)
h = 1.0 / (W - 1)
sp = dict(alpha=8.0 / h * 0.1, beta=1.0, radius=R, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25, rho=0.5, gamma=0.5,
          kappa=1.0, tau=0.0, sigma=0.0, theta=1.0, iters_per_round=1, rounds=1)
ex_lo = max(2.0, 2.0 / (R * h) ** 2)  # supports fit the window: the window sum is the all-pairs sum
eps = np.stack([np.full(M, 4 * ex_lo), np.full(M, 57.0)], axis=1)
with msa.Solver(msa.Params.from_solver(1, H, W, C, sp), I[None]) as s:
    d = msa.DalParams(steps=M, iters=0, ex_lo=ex_lo)
    s.dal(d, eps)  # warm-up
    t0 = time.perf_counter()
    s.dal(d, eps)
    t_cost = time.perf_counter() - t0
    t0 = time.perf_counter()
    J, g = s.dal_gradient(d, eps)
    t_grad = time.perf_counter() - t0
    d2 = msa.DalParams(steps=M, iters=iters, sigma0=1e4, ex_lo=ex_lo)
    t0 = time.perf_counter()
    e, Jh, sh = s.dal(d2, eps)
    t_dal = time.perf_counter() - t0
    n_off = s.query().window_size - 1
print(json.dumps({"H": H, "W": W, "R": R, "M": M, "window_offsets": n_off, "ex_lo": ex_lo,
                  "cost_eval_s": t_cost, "gradient_s": t_grad, "dal_iters": iters, "dal_s": t_dal,
                  "J": [float(x) for x in Jh], "sigma": [float(x) for x in sh],
                  "forward_terms_per_s": H * W * n_off * M / t_cost}), flush=True)
