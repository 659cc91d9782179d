"""Subprocess helper for kernel-variant tests: runs one case through the C ABI and saves the
fields. The kernel variant is chosen by the environment of the process (MSA_K1 = sweep | tile | generic)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_16154_b200 as msa  # noqa: E402


def main():
    spec = json.loads(sys.argv[1])
    out = sys.argv[2]
    rng = np.random.default_rng(spec["seed"])
    B, H, W, C = spec["shape"]
    I = rng.random((B, H, W, C), dtype=np.float32)
    sp = spec["params"]
    p = msa.Params(batch=B, height=H, width=W, channels=C, **sp)
    res = {}
    with msa.Solver(p, I) as s:
        if spec.get("random_state", True):
            c = np.clip(I + 0.05 * rng.standard_normal(I.shape).astype(np.float32), 0, 1)
            s.set_field(msa.FIELD_C, c)
            s.set_field(msa.FIELD_CBAR, np.clip(c + 0.02 * rng.standard_normal(I.shape).astype(np.float32), 0, 1))
            s.set_field(msa.FIELD_P, (0.3 * rng.standard_normal((B, H, W, 2 * C))).astype(np.float32))
            s.set_field(msa.FIELD_MU, (0.3 * rng.standard_normal((B, H, W, 2 * C))).astype(np.float32))
        s.step(spec["iters"])
        for name, f in (("c", msa.FIELD_C), ("cbar", msa.FIELD_CBAR), ("p", msa.FIELD_P), ("mu", msa.FIELD_MU)):
            res[name] = s.get_field(f)
    np.savez(out, **res)


if __name__ == "__main__":
    main()
