"""World-size-2 `gloo` test of the row-slab path on CPU: the library's row
partition (msa_partition_rows) and halo plan (msa_halo_plan) - the same plan the driver issues as
NCCL send/recv on the GPU - drive an exchange between two processes that each iterate their slab
(plus ghost rows) with the oracle. The gathered slabs must equal the single-process run bitwise
(P19), and the all-reduced per-slab sums must equal the whole-image sums."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2510_16154_b200 as msa

H, W, C, R, K, ROUNDS = 31, 19, 3, 3, 4, 2


def _params(h, w):
    hh = 1.0 / (W - 1)
    return oracle.Params(height=h, width=w, channels=C, radius=R, hx=1.0 / (W - 1), hy=1.0 / (H - 1), eps_c=57.0,
                         dt=0.25, alpha=8.0 / hh, beta=1.0, rho=2.5 * hh, gamma=2.5 * hh, iters_per_round=K,
                         rounds=ROUNDS)


def _image():
    return np.random.default_rng(42).random((H, W, C))


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    msa.build()
    r0, nr, G = msa.partition_rows(H, world, rank, R)
    lo, hi = max(0, r0 - G), min(H, r0 + nr + G)
    I = _image()
    st = oracle.State(_params(hi - lo, W), I[lo:hi])
    fields = {msa.FIELD_C: "c", msa.FIELD_CBAR: "cbar", msa.FIELD_P: "p", msa.FIELD_MU: "mu"}

    def exchange(phase):
        reqs, recvs = [], []
        for field, peer, send, row0, n in msa.halo_plan(H, world, rank, R, phase):
            arr = getattr(st, fields[field])
            block = arr[row0 - lo:row0 - lo + n]
            if send:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(block)), peer))
            else:
                buf = torch.empty(block.shape, dtype=torch.float64)
                reqs.append(dist.irecv(buf, peer))
                recvs.append((arr, row0 - lo, n, buf))
        for r in reqs:
            r.wait()
        for arr, a, n, buf in recvs:
            arr[a:a + n] = buf.numpy()

    mu_dirty = True
    sums = []
    for it in range(K * ROUNDS):
        if mu_dirty:
            exchange(msa.HALO_MU)
            mu_dirty = False
        exchange(msa.HALO_ITER)
        st.iteration()
        if (it + 1) % K == 0:
            exchange(msa.HALO_ROUND)
            own = st.c[r0 - lo:r0 - lo + nr]
            t = torch.from_numpy(own.reshape(-1, C).sum(0).copy())
            dist.all_reduce(t)
            sums.append(t.numpy().copy())
            st.round_update()
            mu_dirty = True
    own = {k: torch.from_numpy(np.ascontiguousarray(getattr(st, k)[r0 - lo:r0 - lo + nr])) for k in ("c", "cbar", "p", "mu")}
    if rank == 0:
        parts = {k: [own[k]] for k in own}
        for src in range(1, world):
            n_src = msa.partition_rows(H, world, src, R)[1]
            for k in own:
                buf = torch.empty((n_src,) + tuple(own[k].shape[1:]), dtype=torch.float64)
                dist.recv(buf, src)
                parts[k].append(buf)
        np.savez(out_path, sums=np.array(sums), **{k: torch.cat(v).numpy() for k, v in parts.items()})
    else:
        for k in ("c", "cbar", "p", "mu"):
            dist.send(own[k], 0)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world", [2, 3])
def test_row_slabs_match_single_process(world, tmp_path):
    out = str(tmp_path / "dist.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    ref = oracle.State(_params(H, W), _image())
    ref_sums = []
    for it in range(K * ROUNDS):
        ref.iteration()
        if (it + 1) % K == 0:
            ref_sums.append(ref.c.reshape(-1, C).sum(0))
            ref.round_update()
    for k in ("c", "cbar", "p", "mu"):
        assert np.array_equal(res[k], getattr(ref, k)), k
    assert np.allclose(res["sums"], np.array(ref_sums), rtol=1e-13, atol=0)
