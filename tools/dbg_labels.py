import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.environ.get('GRAFT_REPO_ROOT', '.'))
import numpy as np, torch
import paper_2510_16154_b200 as msa, synth, oracle
cfg = synth.CONFIGS['cfg4']; img = synth.generate(cfg.recipe); sp = synth.solver_params(cfg)
B,H,W,C = img.shape
with msa.Solver(msa.Params.from_solver(B,H,W,C,sp), img) as s:
    s.solve(); c0 = s.get_field(msa.FIELD_C)[0]
    for t in range(2):
        lab, cnt, _ = s.labels(0.1); print('gpu', t, cnt, flush=True)

olab, ocnt, _ = oracle.labels(c0, 0.1); print('oracle', ocnt)
print('agree', np.mean(olab == lab[0]))
