"""msa_solve latency with and without the CUDA-graph replay (MSA_NO_GRAPH): the small BASELINE
configs are launch-bound. Each run: reset + 2 warm-up solves (the first one captures), then `reps`
timed reset+solve pairs, host clock around each (msa_solve returns after a stream synchronise).
Prints one JSON line per config and mode. Usage: python tools/time_graph.py [cfg1 cfg2 ...]"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(name, reps):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2510_16154_b200 as msa
    import synth
    cfg = synth.CONFIGS[name]
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    dev = torch.from_numpy(img).cuda()
    with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
        for _ in range(2):
            s.reset(dev)
            s.solve()
        ts = []
        for _ in range(reps):
            s.reset(dev)
            s.sync()
            t0 = time.perf_counter()
            s.solve()
            ts.append(time.perf_counter() - t0)
        launches = s.query().launches
    ts.sort()
    med = ts[len(ts) // 2] * 1e3
    print(json.dumps({"config": name, "graph": "MSA_NO_GRAPH" not in os.environ, "iters": cfg.iters,
                      "solve_ms_median": med, "solve_ms_min": ts[0] * 1e3, "us_per_iter": med * 1e3 / cfg.iters,
                      "px_it_per_s": B * H * W * cfg.iters / (med * 1e-3), "launches_total": launches}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        sys.exit(0)
    names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]
    for name in names:
        for graph in (False, True):
            env = dict(os.environ, MSA_LIB=os.environ.get("MSA_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_16154_b200", "libmsa_testing.so")))
            env.pop("MSA_NO_GRAPH", None)
            if not graph:
                env["MSA_NO_GRAPH"] = "1"
            reps = "50" if name in ("cfg1", "cfg2") else "5"
            subprocess.run([sys.executable, os.path.abspath(__file__), "--child", name, reps], check=True, env=env)
