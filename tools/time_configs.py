"""Times msa_solve on each BASELINE config (device-resident image, CUDA events, after a warm-up
solve) and prints one JSON line per config: ms per iteration, px-it/s, K1 share, HBM fraction."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402

args = [a for a in sys.argv[1:] if "=" not in a]
opts = dict(a.split("=", 1) for a in sys.argv[1:] if "=" in a)  # e.g. scheme=1
names = args or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for name in names:
    cfg = synth.CONFIGS[name]
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    if "scheme" in opts:
        sp = dict(sp, scheme=int(opts["scheme"]), tau=0.0)
    B, H, W, C = img.shape
    dev = torch.from_numpy(img).cuda()
    with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
        s.solve()
        s.reset(dev)
        s.set_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.solve()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        t = s.get_timing()
        l0 = torch.cuda.Event(enable_timing=True)
        l1 = torch.cuda.Event(enable_timing=True)
        l0.record()
        lab, cnt, _ = s.labels(cfg.delta_label)
        l1.record()
        torch.cuda.synchronize()
    npx = B * H * W
    k1 = t["iter_ms"] / max(t["iter_launches"], 1)
    print(json.dumps({"config": name, "scheme": int(opts.get("scheme", 0)), "shape": [B, H, W, C], "iters": cfg.iters, "solve_ms": ms,
                      "ms_per_iter": ms / cfg.iters, "px_it_per_s": npx * cfg.iters / (ms * 1e-3),
                      "k1_ms": k1, "k1_hbm_frac": (28 if int(opts.get("scheme", 0)) == 1 else 44) * C * npx / (k1 * 1e-3) / 1e9 / peak,
                      "round_ms": t["round_ms"] / max(t["round_launches"], 1), "labels_ms": l0.elapsed_time(l1),
                      "clusters": [int(x) for x in cnt[:4]]}), flush=True)
