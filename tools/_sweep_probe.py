"""Debug probe: run small cases through the sweep kernel in subprocesses, report crash / max diff vs generic."""
import json, os, subprocess, sys
import numpy as np
HERE = os.path.dirname(os.path.abspath(__file__))
RUN = os.path.join(os.path.dirname(HERE), "tests", "_run_case.py")
cases = [((1, 64, 32, 3), 5), ((1, 37, 29, 3), 3), ((1, 64, 64, 3), 3), ((1, 64, 64, 3), 2), ((1, 64, 64, 3), 4),
         ((1, 130, 97, 3), 5), ((1, 16, 16, 3), 3)]
for shape, R in cases:
    B, H, W, C = shape
    h = 1.0 / (W - 1)
    spec = dict(seed=H * 1000 + W + R, shape=list(shape), iters=1,
                params=dict(alpha=8.0 / h, beta=1.0, radius=R, kernel=0, eps_c=20.0, dt=0.25, rho=2.5 * h,
                            gamma=2.5 * h, iters_per_round=2, rounds=1))
    outs = {}
    for v in ("generic", os.environ.get("PROBE_VARIANT", "sweep")):
        env = dict(os.environ, MSA_K1=v)
        out = f"/tmp/probe_{v}.npz"
        r = subprocess.run([sys.executable, RUN, json.dumps(spec), out], env=env, capture_output=True, text=True, timeout=120)
        if r.returncode != 0:
            outs[v] = r.stderr.strip().splitlines()[-1][:200]
        else:
            outs[v] = np.load(out)
    vv = os.environ.get("PROBE_VARIANT", "sweep")
    if isinstance(outs[vv], str) or isinstance(outs["generic"], str):
        print(shape, R, "FAIL", outs[vv] if isinstance(outs[vv], str) else outs["generic"], flush=True)
        continue
    a, b = outs["generic"], outs[vv]
    d = np.abs(a["c"] - b["c"])
    idx = np.unravel_index(np.argmax(d), d.shape)
    print(shape, R, "c maxdiff", float(d.max()), "at", idx, "p eq", bool(np.array_equal(a["p"], b["p"])),
          "rows with diff>1e-6:", sorted(set(np.nonzero(d.max(axis=(0, 2, 3)) > 1e-6)[0].tolist()))[:20],
          "cols:", sorted(set(np.nonzero(d.max(axis=(0, 1, 3)) > 1e-6)[0].tolist()))[:20], flush=True)
