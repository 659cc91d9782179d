"""Write full-size, full-length oracle references for BASELINE.json's five configs (and a 1024^2
cfg4-recipe case that exercises the P = 4 tiles over all 10 rounds) to tests/golden/.

ORACLE-ONLY: this script imports `synth` (the seeded input generator, no method arithmetic) and
`oracle` (the fp64 CPU implementation of SURVEY.md §8(c)); it never loads the CUDA library. Every
stored value comes from `oracle/` (Alg. 2, in the fused reading R1).

Per image it stores (tests/golden/full_<case>.npz):
  input_sha256   hash of the float32 input [B][H][W][C] the generator drew (so the GPU test knows it
                 runs on the same image)
  idx            sampled pixel indices (j, i): the four corners, points on each border, 4096 uniform
  c              the oracle's final colour field at those pixels (fp64; fp32 for batches) [B][n][C]
  stats          the round records (pre-update mu) [B][rounds][8 + C]
  labels         Q(c; delta) of the oracle's final field rounded to fp32 (reading R16), full map
                 [min(B, 4)][H][W] (uint16 when the count allows it)
  labels_sampled (batches) the labels at idx for every image [B][n]
  count          cluster counts [B]
  margin         R17's decision margin of Q on the oracle field: min |d - delta| over the
                 neighbour comparisons of stage (i) [B]

Usage: python tools/make_fullsize_golden.py [case ...]   (cases: cfg1 cfg2 cfg3 cfg4 cfg5 cfg4_1024)
Runs on every host core (OpenMP inside the oracle). Approximate cost on 8 cores: cfg1-2 < 1 min,
cfg4_1024 ~4 min, cfg3 ~12 min, cfg4 ~50 min, cfg5 ~70 min.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
N_UNIFORM = 4096
FULL_MAPS = 4  # full label maps stored per case (the rest sampled: keeps the files small)


def cases() -> dict:
    c = dict(synth.CONFIGS)
    c["cfg4_1024"] = synth.resized(synth.CONFIGS["cfg4"], 1024, 1024)
    return c


def sample_indices(name: str, H: int, W: int) -> np.ndarray:
    rng = np.random.default_rng(int.from_bytes(hashlib.sha256(name.encode()).digest()[:4], "little"))
    pts = [(0, 0), (0, W - 1), (H - 1, 0), (H - 1, W - 1)]
    for t in np.linspace(0, 1, 9)[1:-1]:
        pts += [(0, int(t * (W - 1))), (H - 1, int(t * (W - 1))), (int(t * (H - 1)), 0), (int(t * (H - 1)), W - 1)]
    n = min(N_UNIFORM, H * W)
    flat = rng.choice(H * W, size=n, replace=False)
    pts += [(int(f // W), int(f % W)) for f in flat]
    idx = np.unique(np.array(pts, dtype=np.int64), axis=0)
    return idx


def stage1_margin(c32: np.ndarray, delta: float) -> float:
    """min over 4-neighbour pairs of | ||c_a - c_b||_inf - delta | in fp32 (R16 stage (i), R17)."""
    c = c32.astype(np.float32)
    dx = np.max(np.abs(c[:, 1:] - c[:, :-1]), axis=-1)
    dy = np.max(np.abs(c[1:, :] - c[:-1, :]), axis=-1)
    d = np.float32(delta)
    return float(min(np.min(np.abs(dx - d)), np.min(np.abs(dy - d))))


def make(name: str, cfg) -> dict:
    img = synth.generate(cfg.recipe)
    sp = synth.solver_params(cfg)
    B, H, W, C = img.shape
    idx = sample_indices(name, H, W)
    prm = oracle.Params.from_solver(H, W, C, sp)
    out_c = np.zeros((B, len(idx), C))
    out_stats = np.zeros((B, cfg.rounds, oracle.NSTAT_FIXED + C))
    labs, counts, margins = [], [], []
    t0 = time.time()
    for b in range(B):
        st = oracle.State(prm, img[b].astype(np.float64))
        st.run(cfg.iters)
        out_c[b] = st.c[idx[:, 0], idx[:, 1]]
        out_stats[b] = np.array(st.stats[:cfg.rounds])
        c32 = st.c.astype(np.float32)
        lab, cnt, _ = oracle.labels(c32, cfg.delta_label)
        labs.append(lab)
        counts.append(cnt)
        margins.append(stage1_margin(c32, cfg.delta_label))
        print(f"{name} image {b + 1}/{B}: count {cnt}, margin {margins[-1]:.3g}, {time.time() - t0:.0f} s",
              flush=True)
    lab = np.stack(labs)
    lab = lab.astype(np.uint16) if lab.max() < 65535 else lab
    path = os.path.join(GOLDEN, f"full_{name}.npz")
    extra = {}
    if B > FULL_MAPS:  # batches: full label maps of the first FULL_MAPS images, sampled labels of all
        extra["labels_sampled"] = np.stack([lab[b][idx[:, 0], idx[:, 1]] for b in range(B)])
        lab = lab[:FULL_MAPS]
        out_c = out_c.astype(np.float32)  # 6e-8 relative rounding against the 1e-4 gate; 4x smaller
    np.savez_compressed(path, input_sha256=np.frombuffer(hashlib.sha256(img.tobytes()).digest(), np.uint8),
                        idx=idx, c=out_c, stats=out_stats, labels=lab, count=np.array(counts, np.int32),
                        margin=np.array(margins), iters=np.int64(cfg.iters), rounds=np.int64(cfg.rounds), **extra)
    meta = dict(case=name, shape=[B, H, W, C], iters=cfg.iters, rounds=cfg.rounds, counts=counts,
                margin_min=min(margins), oracle_seconds=round(time.time() - t0, 1), cores=os.cpu_count(),
                bytes=os.path.getsize(path))
    print(json.dumps(meta), flush=True)
    return meta


def main(argv) -> None:
    oracle.build()
    synth.build()
    cs = cases()
    names = argv or ["cfg1", "cfg2", "cfg4_1024", "cfg3", "cfg4", "cfg5"]
    log = os.path.join(GOLDEN, "full_provenance.jsonl")
    for n in names:
        meta = make(n, cs[n])
        with open(log, "a") as f:
            f.write(json.dumps(meta) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:])
