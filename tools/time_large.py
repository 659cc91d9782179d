"""Per-iteration time of the large-support path (NEXT-3) vs the generic kernel on a synthetic
image: device-resident, CUDA events around msa_step batches. Prints interaction terms per second
and the FP32 lane-operation rate (15 FMA-pipe operations per pixel-offset term, ordered form).
usage: python tools/time_large.py H W R [iters]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402

H, W, R = (int(a) for a in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 50
rng = np.random.default_rng(0)
img = torch.from_numpy(rng.random((1, H, W, 3), dtype=np.float32)).cuda()
h = 1.0 / (W - 1)
p = msa.Params(batch=1, height=H, width=W, channels=3, alpha=8.0 / h, beta=1.0, radius=R, eps_c=57.0, dt=0.25,
               rho=2.5 * h, gamma=2.5 * h, iters_per_round=iters, rounds=1)
with msa.Solver(p, img) as s:
    s.step(iters)
    s.sync()
    s.set_timing(True)  # CUDA events on the library's stream around the iteration batches
    s.step(iters)
    s.sync()
    t = s.get_timing()
    ms = t["iter_ms"] / max(t["iter_launches"], 1)
    n_off = s.query().active_offsets
terms = H * W * n_off
print(json.dumps({"H": H, "W": W, "R": R, "variant": os.environ.get("MSA_K1", "default"), "ms_per_iter": ms,
                  "active_offsets": n_off, "terms_per_s": terms / (ms * 1e-3),
                  "fp32_T_lane_ops": 15 * terms / (ms * 1e-3) / 1e12}), flush=True)
