"""One bench step (reset + solve + labels) of a BASELINE config, for the ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
cfg = synth.CONFIGS[name]
img = synth.generate(cfg.recipe)
sp = synth.solver_params(cfg)
B, H, W, C = img.shape
dev = torch.from_numpy(img).cuda()
with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
    s.reset(dev)
    s.solve()
    lab, cnt, _ = s.labels(cfg.delta_label)
print("ok", name, "clusters", list(cnt))
