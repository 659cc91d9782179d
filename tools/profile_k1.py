"""Runs a few fused iterations of a BASELINE config through the C ABI (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 5
opts = dict(a.split("=", 1) for a in sys.argv[3:] if "=" in a)  # e.g. scheme=1
cfg = synth.CONFIGS[name]
img = synth.generate(cfg.recipe)
sp = synth.solver_params(cfg)
if "scheme" in opts:
    sp = dict(sp, scheme=int(opts["scheme"]), tau=0.0)
B, H, W, C = img.shape
with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), torch.from_numpy(img).cuda()) as s:
    s.step(iters)
    s.sync()
print("ok", name, iters)
