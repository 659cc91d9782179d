"""Times the fp64 CPU oracle (as it stands) on every BASELINE config (SURVEY §8(d) "oracle timing":
all five configs, plus single-thread times for configs 1-2), on the host it runs on. Each
measurement is a bounded sample: the bottom-left crop of image 0 with the full image's spacing
and parameters, a fixed iteration count, repeated until ~budget seconds. One JSON line per
(config, threads). Usage: python tools/time_oracle.py [budget_s]"""
import json
import os
import subprocess
import sys
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAMPLES = {"cfg1": (64, 200), "cfg2": (256, 50), "cfg3": (256, 50), "cfg4": (256, 50), "cfg5": (128, 50)}


def child(name, budget):
    sys.path.insert(0, ROOT)
    import numpy as np
    import oracle
    import synth
    cfg = synth.CONFIGS[name]
    img = synth.generate(replace(cfg.recipe, batch=1))
    sp = synth.solver_params(cfg)
    H, W, C = img.shape[1:]
    side, iters = SAMPLES[name]
    crop = img[0, :side, :side].astype(np.float64)
    prm = oracle.Params.from_solver(side, side, C, sp)
    prm.hx, prm.hy = 1.0 / (W - 1), 1.0 / (H - 1)
    prm.iters_per_round = iters
    done, t0 = 0, time.perf_counter()
    while True:
        s = oracle.State(prm, crop)
        s.run(iters)
        done += 1
        el = time.perf_counter() - t0
        if el >= budget or done >= 200:
            break
    rate = done * side * side * iters / el
    print(json.dumps({"config": name, "threads": int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)),
                      "px_it_per_s": rate, "sample": f"{side}x{side} crop of image 0 ({H}x{W}x{C}), R={sp['radius']}, "
                      f"{iters} iterations x {done}", "seconds": el,
                      "full_config_estimate_s": cfg.recipe.batch * H * W * cfg.iters / rate}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--child":
        child(sys.argv[2], float(sys.argv[3]))
        sys.exit(0)
    budget = sys.argv[1] if len(sys.argv) > 1 else "8"
    sys.path.insert(0, ROOT)
    import oracle
    oracle.build()
    runs = [(n, None) for n in SAMPLES] + [("cfg1", 1), ("cfg2", 1)]
    for name, threads in runs:
        env = dict(os.environ)
        if threads:
            env["OMP_NUM_THREADS"] = str(threads)
        else:
            env.pop("OMP_NUM_THREADS", None)
        subprocess.run([sys.executable, os.path.abspath(__file__), "--child", name, budget], check=True, env=env)
