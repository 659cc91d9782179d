"""Subprocess helper for the row-slab test (run with MSA_NCCL_LOOPBACK=1): one context on the
whole image, then `world` contexts of a row-slab world (shard = rows), each driven by its own
thread and connected by the library's in-process loopback transport. Checks that the slabs
reassemble the one-context fields bitwise, that labels / counts / palettes are identical, and that
the round records agree (fp64 sums over slabs: 1e-9 relative). Prints one JSON line."""
import json
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2510_16154_b200 as msa  # noqa: E402

FIELDS = (("c", msa.FIELD_C), ("cbar", msa.FIELD_CBAR), ("p", msa.FIELD_P), ("mu", msa.FIELD_MU))
STAT_KEYS = ("round", "iters", "e_tv", "e_fid", "primal", "dual", "gap", "al_residual")


def image(rng, B, H, W, C):
    # piecewise-constant blocks (so the labels have structure) + noise
    by, bx = max(H // 5, 1), max(W // 4, 1)
    cols = rng.random((B, H // by + 1, W // bx + 1, C))
    yy, xx = np.meshgrid(np.arange(H) // by, np.arange(W) // bx, indexing="ij")
    I = cols[:, yy, xx, :] + 0.05 * rng.standard_normal((B, H, W, C))
    return np.clip(I, 0, 1).astype(np.float32)


def run_one(p, I, delta, max_k):
    with msa.Solver(p, I) as s:
        st = s.solve()
        info = s.query()
        f = {k: s.get_field(w) for k, w in FIELDS}
        lab, cnt, pal = s.labels(delta, max_k)
        return dict(row0=info.row0, nrows=info.nrows, image0=info.image0, nimages=info.nimages, stats=st, fields=f,
                    lab=lab, cnt=cnt, pal=pal, launches=info.launches)


def check_batch(spec, base, I, ref, delta, max_k, world):
    # images split across ranks, no collective: each rank's images equal the one-context run's
    out = [run_one(msa.Params(**base, shard=msa.SHARD_BATCH, world=world, rank=r), I, delta, max_k)
           for r in range(world)]
    assert sum(o["nimages"] for o in out) == I.shape[0]
    for o in out:
        sl = slice(o["image0"], o["image0"] + o["nimages"])
        for k, _ in FIELDS:
            assert np.array_equal(o["fields"][k], ref["fields"][k][sl]), ("batch", world, k)
        assert np.array_equal(o["lab"], ref["lab"][sl]) and np.array_equal(o["cnt"], ref["cnt"][sl])
        assert np.array_equal(o["pal"], ref["pal"][sl])
    return {"fields": "bitwise", "labels": "identical", "images": [o["nimages"] for o in out]}


def main():
    spec = json.loads(sys.argv[1])
    B, H, W, C = spec["shape"]
    rng = np.random.default_rng(spec["seed"])
    I = image(rng, B, H, W, C)
    base = dict(batch=B, height=H, width=W, channels=C, **spec["params"])
    delta, max_k = spec.get("delta", 0.1), 64
    ref = run_one(msa.Params(**base), I, delta, max_k)
    report = {"shape": spec["shape"], "worlds": {}}
    if spec.get("shard") == "batch":
        for world in spec["worlds"]:
            report["worlds"][str(world)] = check_batch(spec, base, I, ref, delta, max_k, world)
        print(json.dumps(report), flush=True)
        return
    for world in spec["worlds"]:
        nid = msa.nccl_unique_id()
        out = [None] * world
        err = [None] * world

        def work(r):
            try:
                p = msa.Params(**base, shard=msa.SHARD_ROWS, world=world, rank=r, nccl_id=nid)
                out[r] = run_one(p, I, delta, max_k)
            except Exception as e:  # reported below
                err[r] = repr(e)

        ts = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not any(err), err
        # slabs tile the image in rank order
        assert [o["row0"] for o in out] == sorted(o["row0"] for o in out)
        assert sum(o["nrows"] for o in out) == H and out[0]["row0"] == 0
        for k, _ in FIELDS:
            got = np.concatenate([o["fields"][k] for o in out], axis=1)
            diff = float(np.max(np.abs(got - ref["fields"][k])))
            assert np.array_equal(got, ref["fields"][k]), (world, k, diff)
        lab = np.concatenate([o["lab"] for o in out], axis=1)
        assert np.array_equal(lab, ref["lab"]), (world, "labels", int(np.sum(lab != ref["lab"])))
        for o in out:
            assert np.array_equal(o["cnt"], ref["cnt"]), (world, "counts", o["cnt"], ref["cnt"])
            assert np.array_equal(o["pal"], ref["pal"]), (world, "palette")
        worst = 0.0
        for o in out:
            assert len(o["stats"]) == len(ref["stats"])
            for a, b in zip(o["stats"], ref["stats"]):
                assert a["round"] == b["round"] and a["iters"] == b["iters"]
                for k in STAT_KEYS[2:]:
                    den = max(abs(b[k]), 1e-30)
                    rel = abs(a[k] - b[k]) / den
                    worst = max(worst, rel)
                    assert rel <= 1e-9 or abs(a[k] - b[k]) <= 1e-12, (world, k, a[k], b[k])
        report["worlds"][str(world)] = {"fields": "bitwise", "labels": "identical", "clusters": ref["cnt"].tolist(),
                                        "stats_max_rel": worst, "launches": [o["launches"] for o in out]}
    print(json.dumps(report), flush=True)


if __name__ == "__main__":
    main()
