"""Convergence per time of the two iteration schemes (msa.h MSA_SCHEME_*) on one BASELINE recipe:
per round, the ROF energy K = E_TV + E_fid of c, the round record's gap and residual, and the
device time so far (CUDA events). dt=0 isolates the optimiser (the ROF problem, where both
schemes converge to the same minimiser); the default dt adds the agent dynamics.
usage: python tools/compare_schemes.py cfg3 [H W] [dt=0] [rounds=10] [K=100]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402

pos = [a for a in sys.argv[1:] if "=" not in a]
opts = dict(a.split("=", 1) for a in sys.argv[1:] if "=" in a)
name = pos[0] if pos else "cfg3"
cfg = synth.CONFIGS[name]
if len(pos) >= 3:
    cfg = synth.resized(cfg, int(pos[1]), int(pos[2]))
rounds = int(opts.get("rounds", cfg.rounds))
K = int(opts.get("K", cfg.iters_per_round))
cfg = synth.resized(cfg, cfg.recipe.height, cfg.recipe.width, rounds=1, iters_per_round=K)
img = synth.generate(cfg.recipe)
B, H, W, C = img.shape
dev = torch.from_numpy(img).cuda()
for scheme in (0, 1):
    sp = dict(synth.solver_params(cfg), scheme=scheme, tau=0.0)
    if "dt" in opts:
        sp["dt"] = float(opts["dt"])
    with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
        s.solve()  # warm-up (one round)
        s.reset(dev)
        t_ms = 0.0
        for r in range(rounds):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = s.solve()[-1]
            e1.record()
            torch.cuda.synchronize()
            t_ms += e0.elapsed_time(e1)
            print(json.dumps({"config": name, "shape": [B, H, W, C], "dt": sp["dt"], "scheme": scheme, "round": r,
                              "iters": (r + 1) * K, "time_ms": round(t_ms, 3),
                              "K_energy": st["e_tv"] + st["e_fid"], "gap": st["gap"],
                              "residual": st["al_residual"]}), flush=True)
