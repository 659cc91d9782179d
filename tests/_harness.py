"""Shared test helpers: run the CUDA path (through the C ABI binding) and the oracle on the
same seeded inputs, and the parity metric of SURVEY.md §8(c) R17."""
from __future__ import annotations

import os

import numpy as np

import oracle
import synth


def rel_err_per_pixel(c_gpu: np.ndarray, c_ref: np.ndarray) -> np.ndarray:
    """R17: e(n) = ||c_gpu(n) - c_ref(n)||_inf / max(||c_ref(n)||_inf, 1e-3), per pixel."""
    num = np.max(np.abs(c_gpu.astype(np.float64) - c_ref), axis=-1)
    den = np.maximum(np.max(np.abs(c_ref), axis=-1), 1e-3)
    return num / den


def oracle_params(H: int, W: int, C: int, sp: dict, **over) -> oracle.Params:
    p = oracle.Params.from_solver(H, W, C, sp)
    for k, v in over.items():
        setattr(p, k, v)
    return p


def run_oracle(image: np.ndarray, sp: dict, n_iters: int | None = None, **over):
    """image float32 [B][H][W][C] -> list of oracle States (one per image) after n_iters iterations."""
    B, H, W, C = image.shape
    p = oracle_params(H, W, C, sp, **over)
    n = n_iters if n_iters is not None else p.rounds * p.iters_per_round
    out = []
    for b in range(B):
        s = oracle.State(p, image[b].astype(np.float64))
        s.run(n)
        out.append(s)
    return out


def gpu_params(image: np.ndarray, sp: dict, **over):
    import paper_2510_16154_b200 as msa
    B, H, W, C = image.shape
    p = msa.Params.from_solver(B, H, W, C, sp)
    for k, v in over.items():
        setattr(p, k, v)
    return p


def config_case(name: str, H: int | None = None, W: int | None = None, B: int | None = None,
                rounds: int | None = None, iters_per_round: int | None = None):
    cfg = synth.CONFIGS[name]
    if H is not None or W is not None or B is not None or rounds is not None or iters_per_round is not None:
        cfg = synth.resized(cfg, H or cfg.recipe.height, W or cfg.recipe.width, batch=B, rounds=rounds,
                            iters_per_round=iters_per_round)
    img = synth.generate(cfg.recipe)
    return cfg, img, synth.solver_params(cfg)


TESTING_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_16154_b200",
                           "libmsa_testing.so")


def hook_env(**hooks) -> dict:
    """Environment of a subprocess that runs the testing build of the library (the same kernels plus the
    environment test hooks, the experimental sweep K1 and the in-process NCCL transport):
    the product libmsa.so reads no environment variable, so hook-driven cases must load this one."""
    env = dict(os.environ, MSA_LIB=os.environ.get("MSA_TEST_LIB", TESTING_LIB))  # MSA_TEST_LIB: a variant build
    env.update({k: str(v) for k, v in hooks.items()})
    return env
