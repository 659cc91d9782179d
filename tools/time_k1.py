"""K1 time per iteration on a BASELINE config (CUDA events through msa_set_timing, after warm-up
iterations): python tools/time_k1.py cfgN [iters] [reps]. Prints one JSON line with the K1 ms, the
HBM fraction of its algorithmic bytes (44 C bytes per pixel-iteration) and the SM
clock sampled while it ran. Load a variant library with MSA_LIB=..."""
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
cfg = synth.CONFIGS[name]
img = synth.generate(cfg.recipe)
sp = synth.solver_params(cfg)
B, H, W, C = img.shape
out = []
with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), torch.from_numpy(img).cuda()) as s:
    s.step(5)
    s.sync()
    for r in range(reps):
        s.set_timing(True)
        clk = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "50"],
                               stdout=subprocess.PIPE, text=True)
        s.step(iters)
        s.sync()
        clk.terminate()
        mhz = [int(v) for v in clk.communicate()[0].split() if v.isdigit()]
        t = s.get_timing()
        s.set_timing(False)
        k1 = t["iter_ms"] / max(t["iter_launches"], 1)
        out.append((k1, sorted(mhz)[len(mhz) // 2] if mhz else None))
npx = B * H * W
k1 = min(v[0] for v in out)
print(json.dumps({"config": name, "lib": os.environ.get("MSA_LIB", "libmsa.so"), "k1_ms": k1,
                  "k1_ms_all": [round(v[0], 4) for v in out], "sm_mhz": [v[1] for v in out],
                  "hbm_frac": 44 * C * npx / (k1 * 1e-3) / 1e9 / peak}), flush=True)
