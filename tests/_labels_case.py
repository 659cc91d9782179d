"""Subprocess helper: solve one synthetic case through the C ABI and save labels, counts, palette.
The labels path is chosen by the environment (MSA_LABELS_PARTS = number of virtual row parts)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_16154_b200 as msa  # noqa: E402
import synth  # noqa: E402


def main():
    spec = json.loads(sys.argv[1])
    cfg = synth.resized(synth.CONFIGS[spec["cfg"]], spec["H"], spec["W"], rounds=spec["rounds"],
                        iters_per_round=spec["K"])
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    with msa.Solver(msa.Params.from_solver(B, H, W, C, sp), img) as s:
        s.solve()
        lab, cnt, pal = s.labels(spec.get("delta", cfg.delta_label), max_k=64)
    np.savez(sys.argv[2], labels=lab, counts=cnt, palette=pal)


if __name__ == "__main__":
    main()
