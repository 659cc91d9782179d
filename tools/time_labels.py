"""Labels timing per BASELINE config after a solve: three device-output calls (the first is cold)
and two host-output calls, wall clock with synchronisation. usage: python tools/time_labels.py cfg2 cfg3"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2510_16154_b200 as msa
import synth
for name in sys.argv[1:]:
    cfg = synth.CONFIGS[name]
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    dev = torch.from_numpy(img).cuda()
    with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), dev) as s:
        s.solve()
        lab = torch.empty((B, H, W), dtype=torch.int32, device="cuda")
        cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
        ts = []
        for i in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            s.labels(cfg.delta_label, 0, out=(lab, cnt, None))
            torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
        ts2 = []
        for i in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            l, c, _ = s.labels(cfg.delta_label)
            ts2.append((time.perf_counter() - t0) * 1e3)
        print(json.dumps({"config": name, "labels_dev_ms": ts, "labels_host_ms": ts2, "clusters": c[:4].tolist()}), flush=True)
