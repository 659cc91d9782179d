"""Seeded synthetic workloads shared by the CUDA harness and the oracle tests.

This module draws images and states the five BASELINE.json configurations; it
holds none of the method's arithmetic (no kernel, stencil or update). Recipes:
SURVEY.md §8(d) "Generator specification" and "Solver parameters"; the images
stand in for the paper's photographs / MRI scan,
which are not available. The C generator (synth.c) is built into
``synth/libmsa_synth.so`` by ``build()`` (also run by ``__graft_entry__.build``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmsa_synth.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class _Recipe(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("channels", ctypes.c_int32), ("kind", ctypes.c_int32), ("n_cells", ctypes.c_int32),
                ("n_clusters", ctypes.c_int32), ("pad_", ctypes.c_int32), ("cluster_sigma", ctypes.c_double),
                ("noise_sigma", ctypes.c_double), ("ramp", ctypes.c_double), ("salt_pepper", ctypes.c_double),
                ("seed", ctypes.c_uint64), ("seed_stride", ctypes.c_uint64)]


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.synth_generate.argtypes = [ctypes.POINTER(_Recipe), ctypes.c_void_p]
        _lib.synth_generate.restype = ctypes.c_int
        _lib.synth_uniform_at.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib.synth_uniform_at.restype = ctypes.c_double
    return _lib


@dataclass(frozen=True)
class Recipe:
    batch: int
    height: int
    width: int
    channels: int
    kind: int  # 0 quadrants, 1 Voronoi
    n_cells: int = 0
    n_clusters: int = 0
    cluster_sigma: float = 0.0
    noise_sigma: float = 0.0
    ramp: float = 0.0
    salt_pepper: float = 0.0
    seed: int = 0
    seed_stride: int = 1


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration: image recipe + solver schedule."""
    name: str
    recipe: Recipe
    radius: int
    rounds: int
    iters_per_round: int
    delta_label: float = 0.1

    @property
    def iters(self) -> int:
        return self.rounds * self.iters_per_round


# BASELINE.json configs[0..4]; counts are totals split into 10 rounds.
CONFIGS = {
    "cfg1": Config("cfg1", Recipe(1, 64, 64, 3, kind=0, noise_sigma=0.05, seed=0), radius=2, rounds=10, iters_per_round=20),
    "cfg2": Config("cfg2", Recipe(1, 512, 512, 3, kind=1, n_cells=16, noise_sigma=0.08, ramp=0.2, seed=1),
                   radius=3, rounds=10, iters_per_round=50),
    "cfg3": Config("cfg3", Recipe(1, 2048, 2048, 3, kind=1, n_cells=64, n_clusters=8, cluster_sigma=0.03,
                                  noise_sigma=0.1, salt_pepper=0.01, seed=2), radius=5, rounds=10, iters_per_round=100),
    "cfg4": Config("cfg4", Recipe(1, 4096, 4096, 3, kind=1, n_cells=128, noise_sigma=0.1, seed=3),
                   radius=5, rounds=10, iters_per_round=100),
    "cfg5": Config("cfg5", Recipe(32, 1024, 1024, 16, kind=1, n_cells=32, noise_sigma=0.05, seed=1000, seed_stride=1),
                   radius=3, rounds=10, iters_per_round=50),
}


def resized(cfg: Config, height: int, width: int, batch: int | None = None, rounds: int | None = None,
            iters_per_round: int | None = None) -> Config:
    """Same recipe at another size (parity cases the oracle finishes in seconds)."""
    rec = replace(cfg.recipe, height=height, width=width, batch=batch if batch is not None else cfg.recipe.batch)
    return replace(cfg, recipe=rec, rounds=rounds if rounds is not None else cfg.rounds,
                   iters_per_round=iters_per_round if iters_per_round is not None else cfg.iters_per_round)


def generate(recipe: Recipe) -> np.ndarray:
    """float32 [B][H][W][C], row 0 = bottom, values in [0,1]."""
    lib = _load()
    r = recipe
    out = np.empty((r.batch, r.height, r.width, r.channels), dtype=np.float32)
    cr = _Recipe(r.batch, r.height, r.width, r.channels, r.kind, r.n_cells, r.n_clusters, 0, r.cluster_sigma,
                 r.noise_sigma, r.ramp, r.salt_pepper, r.seed, r.seed_stride)
    if lib.synth_generate(ctypes.byref(cr), out.ctypes.data) != 0:
        raise ValueError(f"bad recipe {recipe}")
    return out


def uniform_at(seed: int, k: int) -> float:
    return _load().synth_uniform_at(seed, k)


def solver_params(cfg: Config) -> dict:
    """Solver parameters in the paper's Omega = [0,1]^2 units (reading R14).

    Pixel-unit quantities are held fixed across sizes: alpha*h = 8, rho/h = gamma/h = 2.5, with
    h = 1/(W-1). dt = 0.25, eps_c = 57, rho = gamma,
    beta = 1 (eq:cost_TV). eps_x, tau, sigma are left to their documented defaults (<= 0).
    """
    W = cfg.recipe.width
    h = 1.0 / (W - 1) if W > 1 else 1.0
    return dict(alpha=8.0 / h, beta=1.0, radius=cfg.radius, kernel=0, eps_x=0.0, eps_c=57.0, dt=0.25,
                rho=2.5 * h, gamma=2.5 * h, kappa=1.0, tau=0.0, sigma=0.0, theta=1.0,
                iters_per_round=cfg.iters_per_round, rounds=cfg.rounds)
