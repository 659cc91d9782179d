"""K1 time for C = 1..4 channels (cfg4 recipe at 2048^2, R = 5): grey (the paper's own images),
two-channel, RGB and RGBA fields all run on the tiled kernel. usage: [RADIUS=r] python tools/time_channels.py [side] [C,C,...]"""
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2510_16154_b200 as msa
import synth
from dataclasses import replace
SIDE = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
CS = [int(a) for a in sys.argv[2].split(',')] if len(sys.argv) > 2 else [1, 2, 3, 4]
for C in CS:
    cfg = synth.CONFIGS["cfg4"]
    rc = replace(cfg, recipe=replace(cfg.recipe, height=SIDE, width=SIDE, channels=C), rounds=2, iters_per_round=50,
                 radius=int(os.environ.get("RADIUS", cfg.radius)))
    img = synth.generate(rc.recipe)
    sp = synth.solver_params(rc)
    B, H, W, Cc = img.shape
    dev = torch.from_numpy(img).cuda()
    with msa.Solver(msa.Params.from_solver(B, H, W, Cc, sp), dev) as s:
        s.solve(); s.reset(dev); s.set_timing(True); s.solve(); t = s.get_timing()
    k1 = t["iter_ms"] / t["iter_launches"]
    print(json.dumps({"C": C, "shape": [H, W], "k1_ms": k1, "px_it_per_s": H * W / (k1 * 1e-3)}), flush=True)
