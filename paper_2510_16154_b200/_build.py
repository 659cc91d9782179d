"""Builds paper_2510_16154_b200/libmsa.so (all CUDA for sm_100a) with nvcc, in-tree."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libmsa.so")
# the testing library: the same sources with -DMSA_TESTING (environment test hooks) plus
# the experimental pair-symmetric sweep K1 and the in-process NCCL transport; tests and tools load it
# through MSA_LIB. The product library never reads the environment.
TEST_LIB = os.path.join(PKG, "libmsa_testing.so")
SOURCES = ["msa_driver.cu", "msa_kernels.cu", "msa_iter_fast.cu", "msa_iter_cn.cu", "msa_agent_large.cu", "msa_dal.cu",
           "msa_labels.cu"]
TEST_SOURCES = SOURCES + ["msa_iter_sweep.cu", "msa_nccl_loopback.cu"]
FILE_FLAGS: dict[str, list[str]] = {}  # per-file nvcc flags (none at present)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
         "--expt-relaxed-constexpr"]


def _deps() -> list[str]:
    fs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    fs.append(os.path.join(ROOT, "include", "msa.h"))
    return fs


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in _deps())


def build(force: bool = False, verbose: bool = False, defines: tuple = (), lib: str = LIB, build_dir: str = BUILD,
          flags: tuple = (), testing: bool = True) -> str:
    """Builds libmsa.so (and, with testing=True, libmsa_testing.so); returns the product path."""
    if lib == LIB and testing:
        _build_one(force, verbose, ("MSA_TESTING",) + tuple(defines), TEST_LIB, BUILD + "_testing", flags,
                   TEST_SOURCES)
    return _build_one(force, verbose, defines, lib, build_dir, flags, SOURCES if lib == LIB else TEST_SOURCES)


def _build_one(force, verbose, defines, lib, build_dir, flags, sources) -> str:
    if not force and lib in (LIB, TEST_LIB) and not needs_build(lib):
        return lib
    os.makedirs(build_dir, exist_ok=True)
    extra = (["-Xptxas", "-v"] if verbose else []) + [f"-D{d}" for d in defines] + list(flags)

    def compile_one(src: str) -> str:
        obj = os.path.join(build_dir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *FILE_FLAGS.get(src, []), *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(sources)) as ex:
        objs = list(ex.map(compile_one, sources))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
