"""CPU-side checks of the boundary: the sm_100a library loads and exports every symbol that
include/msa.h declares; host-only entry points (validation, workspace sizing, the row
partition) behave as documented. No kernel is launched here."""
import os
import re

import pytest

import paper_2510_16154_b200 as msa

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "msa.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(msa_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    msa.build()
    return msa.lib()


def test_all_declared_symbols_exported(lib):
    decl = _declared_symbols()
    assert len(decl) >= 20
    assert sorted(decl) == sorted(msa.ABI_SYMBOLS)
    for name in decl:
        assert hasattr(lib, name), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", msa.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version(lib):
    assert lib.msa_abi_version() == 3


def _params(**kw):
    base = dict(batch=1, height=64, width=64, channels=3, alpha=504.0, beta=1.0, radius=2, rho=0.04, gamma=0.04,
                iters_per_round=20, rounds=10)
    base.update(kw)
    return msa.Params(**base)


def test_workspace_bytes_formula(lib):
    p = _params(height=100, width=70)
    n = msa.workspace_bytes(p)
    pitch = 96
    fields = 11 * 3 * 100 * pitch * 4
    assert fields <= n <= fields + 4 * 1024 * 1024


@pytest.mark.parametrize("bad", [dict(channels=0), dict(channels=17), dict(alpha=-1.0), dict(beta=-0.1),
                                 dict(radius=256), dict(rho=0.0), dict(gamma=-1.0), dict(kappa=0.0), dict(dt=-0.1),
                                 dict(eps_c=-1.0), dict(iters_per_round=0), dict(rounds=-1), dict(kernel=2),
                                 dict(height=0), dict(world=2, rank=2, shard=1), dict(world=2, shard=0),
                                 dict(tau=1.0, sigma=1.0), dict(alpha=float("nan")), dict(scheme=2),
                                 dict(scheme=1, kappa=1.5), dict(scheme=1, tau=1.0)])
def test_validation_rejects(lib, bad):
    with pytest.raises(msa.MsaError) as e:
        msa.workspace_bytes(_params(**bad)) if "tau" not in bad else _derive_only(bad)
    assert e.value.code == msa.MSA_EINVAL


def _derive_only(bad):
    # tau*sigma*L^2 >= 1 is checked by msa_init (derivation) - exercised through init's validation path
    import ctypes
    import numpy as np
    p = _params(**bad)
    cp, keep = p.c()
    img = np.zeros((1, 64, 64, 3), np.float32)
    ctx = ctypes.c_void_p()
    rc = msa.lib().msa_init(ctypes.byref(cp), img.ctypes.data, 0, None, 0, None, ctypes.byref(ctx))
    msa._check(rc)


def test_partition_rows():
    H, world, R = 4096, 8, 5
    rows = [msa.partition_rows(H, world, r, R) for r in range(world)]
    assert rows[0][0] == 0 and all(g == 5 for _, _, g in rows)
    assert sum(n for _, n, _ in rows) == H
    for a, b in zip(rows, rows[1:]):
        assert a[0] + a[1] == b[0]
    r = [msa.partition_rows(1003, 4, k, 3) for k in range(4)]
    assert [n for _, n, _ in r] == [251, 251, 251, 250]
    assert msa.partition_rows(10, 1, 0, 5) == (0, 10, 0)
    with pytest.raises(msa.MsaError):
        msa.partition_rows(20, 8, 0, 5)  # slabs thinner than the halo


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    with pytest.raises(RuntimeError, match="CUDA"):
        msa.Solver(_params(), np.zeros((1, 64, 64, 3), np.float32))


def test_c_example_builds_against_the_abi():
    """examples/quantize.c compiles and links against include/msa.h + libmsa.so with plain gcc."""
    import __graft_entry__ as g
    exe = g.build_examples()
    assert os.path.exists(exe) and os.access(exe, os.X_OK)


def test_binding_rejects_wrong_buffers():
    """The binding checks dtype and element count before the library sees a pointer (the C ABI
    trusts the sizes it is given)."""
    import numpy as np
    f = msa._ptr_of
    ptr, on_dev, keep = f(np.zeros((2, 3), np.float64), 6, "x")  # inputs are converted
    assert keep.dtype == np.float32 and on_dev == 0
    with pytest.raises(ValueError):
        f(np.zeros(5, np.float32), 6, "x")
    with pytest.raises(TypeError):
        f(np.zeros(6, np.float64), 6, "x", out=True)  # outputs are not converted
    with pytest.raises(TypeError):
        f(np.zeros((3, 4), np.float32)[:, :2], 6, "x", out=True)  # non-contiguous output
    with pytest.raises(TypeError):
        f([0.0] * 6, 6, "x")
    import torch
    with pytest.raises(TypeError):
        f(torch.zeros(6, dtype=torch.float64), 6, "x")
    with pytest.raises(ValueError):
        f(torch.zeros(7), 6, "x")
    assert f(torch.zeros(6), 6, "x")[1] == 0


def test_product_library_reads_no_environment_hook():
    """no environment variable affects numerics. The A/B and test hooks (kernel variant,
    summation order, scaled form, in-process NCCL transport, ...) are compiled only into the testing
    build (-DMSA_TESTING); the product library contains none of their names and neither the
    experimental sweep kernel nor the loopback transport."""
    msa.build()
    prod = open(os.path.join(ROOT, "paper_2510_16154_b200", "libmsa.so"), "rb").read()
    test = open(os.path.join(ROOT, "paper_2510_16154_b200", "libmsa_testing.so"), "rb").read()
    hooks = [b"MSA_K1", b"MSA_NO_SCALED", b"MSA_NCCL_LOOPBACK", b"MSA_LARGE_FROM", b"MSA_LARGE_NOSPLIT",
             b"MSA_DAL_GENERIC", b"MSA_FORCE_GENERIC", b"MSA_LABELS_PARTS", b"MSA_DAL_CHECKPOINT", b"MSA_NO_GRAPH"]
    for h in hooks:
        assert h not in prod, h
        assert h in test, h
    assert b"k_iter_sweep" not in prod and b"k_iter_sweep" in test
    assert b"loopback" not in prod
