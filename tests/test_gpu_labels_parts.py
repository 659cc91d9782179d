"""Labels over row parts (the rows-mode path of msa_labels): stage (i) per part,
segment tables concatenated in row order, one merge, relabel. On one GPU the same path runs on
virtual parts (MSA_LABELS_PARTS); it must reproduce the single-pass rule bit for bit - labels,
counts and palettes - for any number of parts, including one-row parts and more parts than
segments. Cases: the BASELINE recipes at reduced size with their full iteration structure."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
from _harness import hook_env

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(spec, parts, tmp_path):
    out = str(tmp_path / f"lab_{parts}.npz")
    env = hook_env()
    if parts:
        env["MSA_LABELS_PARTS"] = str(parts)
    else:
        env.pop("MSA_LABELS_PARTS", None)
    subprocess.run([sys.executable, os.path.join(HERE, "_labels_case.py"), json.dumps(spec), out], check=True, env=env)
    return np.load(out)


CASES = [
    dict(cfg="cfg1", H=64, W=64, rounds=2, K=10),
    dict(cfg="cfg2", H=96, W=80, rounds=2, K=10),
    dict(cfg="cfg3", H=128, W=128, rounds=2, K=20),          # salt-and-pepper: many small segments
    dict(cfg="cfg3", H=128, W=128, rounds=1, K=1, delta=0.05),  # barely smoothed: thousands of segments
    dict(cfg="cfg5", H=40, W=36, rounds=1, K=5),             # C = 16, batch of images
]


@pytest.mark.parametrize("spec", CASES, ids=lambda s: f"{s['cfg']}_{s['H']}x{s['W']}_{s.get('delta', 'd')}")
def test_parts_equal_single_pass(spec, tmp_path):
    ref = _run(spec, 0, tmp_path)
    for parts in (2, 3, 7, spec["H"]):
        got = _run(spec, parts, tmp_path)
        assert np.array_equal(ref["counts"], got["counts"]), parts
        assert np.array_equal(ref["labels"], got["labels"]), parts
        assert np.array_equal(ref["palette"], got["palette"]), parts
