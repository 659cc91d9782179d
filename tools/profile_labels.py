"""Solve then label one BASELINE config (for an ncu launch list of the labels kernels).
usage: python tools/profile_labels.py cfg3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
img = synth.generate(cfg.recipe)
sp = synth.solver_params(cfg)
B, H, W, C = img.shape
dev = torch.from_numpy(img).cuda()
with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
    s.solve()
    lab = torch.empty((B, H, W), dtype=torch.int32, device="cuda")
    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
    for _ in range(2):
        s.labels(cfg.delta_label, 0, out=(lab, cnt, None))
    torch.cuda.synchronize()
    print("clusters", cnt.tolist()[:4])
