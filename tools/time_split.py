"""Cost of the row-slab overlap structure on one GPU: K1 on one slab-sized image (cfg4 width, H/N
rows, the rows a rank owns at N GPUs) as one launch vs the interior + two boundary launches the
rows mode uses to overlap the halo exchange (MSA_K1_SPLIT=1). Prints one JSON line per (N, mode).
Usage: python tools/time_split.py [N ...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(n):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2510_16154_b200 as msa
    import synth
    cfg = synth.CONFIGS["cfg4"]
    H = cfg.recipe.height // n
    rc = synth.resized(cfg, H, cfg.recipe.width, rounds=2, iters_per_round=100)
    img = synth.generate(rc.recipe)
    sp = synth.solver_params(rc)
    B, H, W, C = img.shape
    dev = torch.from_numpy(img).cuda()
    with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
        s.solve()
        s.reset(dev)
        s.set_timing(True)
        s.solve()
        t = s.get_timing()
    k1 = t["iter_ms"] / max(t["iter_launches"], 1)
    print(json.dumps({"gpus": n, "slab": [H, W], "split": "MSA_K1_SPLIT" in os.environ, "k1_ms": k1,
                      "px_it_per_s": H * W / (k1 * 1e-3)}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(int(sys.argv[2]))
        sys.exit(0)
    for n in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
        for split in (False, True):
            env = dict(os.environ, MSA_LIB=os.environ.get("MSA_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_16154_b200", "libmsa_testing.so")))
            env.pop("MSA_K1_SPLIT", None)
            if split:
                env["MSA_K1_SPLIT"] = "1"
            subprocess.run([sys.executable, os.path.abspath(__file__), "--child", str(n)], check=True, env=env)
