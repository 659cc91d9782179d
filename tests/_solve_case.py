"""Subprocess helper for the CUDA-graph test: a sequence of msa_solve calls (fresh, after a
reset, after msa_step moved the phase inside a round, after set_state) through the C ABI; saves
every field and every round record. MSA_NO_GRAPH in the environment selects direct launches."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_16154_b200 as msa  # noqa: E402

STAT_KEYS = ("round", "iters", "e_tv", "e_fid", "primal", "dual", "gap", "al_residual")


def main():
    spec = json.loads(sys.argv[1])
    out = sys.argv[2]
    rng = np.random.default_rng(spec["seed"])
    B, H, W, C = spec["shape"]
    I = rng.random((B, H, W, C), dtype=np.float32)
    I2 = rng.random((B, H, W, C), dtype=np.float32)
    p = msa.Params(batch=B, height=H, width=W, channels=C, **spec["params"])
    res = {}
    recs = []

    def snap(tag, s, st):
        for name, f in (("c", msa.FIELD_C), ("p", msa.FIELD_P), ("mu", msa.FIELD_MU)):
            res[f"{tag}_{name}"] = s.get_field(f)
        recs.extend([[r[k] for k in STAT_KEYS] for r in st])
        info = s.query()
        res[f"{tag}_info"] = np.array([info.iters_done, info.launches], dtype=np.int64)

    with msa.Solver(p, I) as s:
        snap("a", s, s.solve())            # first solve: captured
        snap("b", s, s.solve())            # continues from the end state (other rho / set)
        s.reset(I2)
        snap("c", s, s.solve())            # same start state as "a": replayed
        s.step(3)                          # phase inside a round
        snap("d", s, s.solve())
        blob = s.get_state()
        s.reset(I)
        snap("e", s, s.solve())
        s.set_state(blob)
        snap("f", s, s.solve())
    res["records"] = np.array(recs, dtype=np.float64)
    np.savez(out, **res)


if __name__ == "__main__":
    main()
