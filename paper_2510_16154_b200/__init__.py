"""Python binding of the msa C ABI (include/msa.h) - argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``libmsa.so`` (sm_100a). There is
no CPU fallback: importing works without a GPU (for ``build()`` and symbol checks), but
creating a :class:`Solver` needs the built library and a CUDA device and fails loudly
otherwise. PyTorch is used only for device memory (the workspace), streams and, in
multi-GPU runs, the process group that broadcasts the NCCL id.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, asdict, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# MSA_LIB: A/B hook for variant builds of the same sources (tools/build_variant.py); default in-tree
LIB_PATH = os.environ.get("MSA_LIB") or os.path.join(_PKG, "libmsa.so")

MSA_OK, MSA_EINVAL, MSA_ENOMEM, MSA_ECUDA, MSA_ENCCL, MSA_EDIVERGED, MSA_ESTATE = 0, -1, -2, -3, -4, -5, -6
SHARD_NONE, SHARD_ROWS, SHARD_BATCH = 0, 1, 2
FIELD_C, FIELD_CBAR, FIELD_P, FIELD_MU, FIELD_I = 0, 1, 2, 3, 4
KERNEL_WENDLAND, KERNEL_PRINTED = 0, 1
SCHEME_CP_ROUNDS, SCHEME_LINEARISED_ADMM = 0, 1

# every symbol include/msa.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ["msa_abi_version", "msa_last_error", "msa_workspace_bytes", "msa_partition_rows",
               "msa_nccl_unique_id", "msa_halo_plan", "msa_init", "msa_reset", "msa_step", "msa_solve",
               "msa_solve_until", "msa_solve_until_balanced", "msa_labels", "msa_label_margin",
               "msa_get_field", "msa_set_field", "msa_get_stats", "msa_state_bytes", "msa_get_state",
               "msa_set_state", "msa_query", "msa_set_timing", "msa_get_timing", "msa_dal", "msa_dal_gradient", "msa_dal_admm",
               "msa_sync", "msa_free"]


class MsaError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"msa error {code}: {msg}")
        self.code = code


class _DalParams(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("cost", ctypes.c_int32), ("iters", ctypes.c_int32),
                ("max_ls", ctypes.c_int32), ("sigma0", ctypes.c_double), ("b", ctypes.c_double),
                ("c", ctypes.c_double), ("ex_lo", ctypes.c_double), ("ex_hi", ctypes.c_double),
                ("ec_lo", ctypes.c_double), ("ec_hi", ctypes.c_double), ("eta", ctypes.c_double),
                ("eta_grad", ctypes.c_double), ("gamma_ls", ctypes.c_int32), ("reserved_", ctypes.c_int32)]


@dataclass
class DalParams:
    """msa_dal_params (include/msa.h): NEXT-1, Algorithm 1 of the paper."""
    steps: int
    cost: int = 0
    iters: int = 10
    max_ls: int = 30
    sigma0: float = 1.0
    b: float = 0.5
    c: float = 1e-4
    ex_lo: float = 2.0
    ex_hi: float = 1100.0
    ec_lo: float = 2.0
    ec_hi: float = 1100.0
    eta: float = 0.0       # Remark 3.4 cost stationarity (1e-10); 0: run `iters` iterations
    eta_grad: float = 0.0  # Remark 3.4 projected-gradient tolerance; 0: off
    gamma_ls: int = 0      # dal_admm: two-way Armijo search for the ascent step (remark after Alg. 2)

    def c_struct(self) -> "_DalParams":
        return _DalParams(**asdict(self), reserved_=0)


class _CParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("channels", ctypes.c_int32), ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("radius", ctypes.c_int32), ("kernel", ctypes.c_int32), ("eps_x", ctypes.c_double),
                ("eps_c", ctypes.c_double), ("dt", ctypes.c_double), ("rho", ctypes.c_double),
                ("gamma", ctypes.c_double), ("kappa", ctypes.c_double), ("tau", ctypes.c_double),
                ("sigma", ctypes.c_double), ("theta", ctypes.c_double), ("iters_per_round", ctypes.c_int32),
                ("rounds", ctypes.c_int32), ("shard", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("device", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("scheme", ctypes.c_int32)]


class RoundStats(ctypes.Structure):
    _fields_ = [("round", ctypes.c_int32), ("images", ctypes.c_int32), ("iters", ctypes.c_int64),
                ("e_tv", ctypes.c_double), ("e_fid", ctypes.c_double), ("primal", ctypes.c_double),
                ("dual", ctypes.c_double), ("gap", ctypes.c_double), ("al_residual", ctypes.c_double),
                ("rho", ctypes.c_double), ("nonfinite", ctypes.c_double), ("mean", ctypes.c_double * 16)]

    def as_dict(self, C: int = 16) -> dict:
        d = {f[0]: getattr(self, f[0]) for f in self._fields_ if f[0] != "mean"}
        d["mean"] = [self.mean[k] for k in range(C)]
        return d


class Info(ctypes.Structure):
    _fields_ = [("row0", ctypes.c_int32), ("nrows", ctypes.c_int32), ("image0", ctypes.c_int32),
                ("nimages", ctypes.c_int32), ("ghost_rows", ctypes.c_int32), ("pitch", ctypes.c_int32),
                ("hx", ctypes.c_double), ("hy", ctypes.c_double), ("eps_x", ctypes.c_double),
                ("tau", ctypes.c_double), ("sigma", ctypes.c_double), ("theta", ctypes.c_double),
                ("window_size", ctypes.c_int32), ("active_offsets", ctypes.c_int32),
                ("iters_done", ctypes.c_int64), ("launches", ctypes.c_int64), ("rho", ctypes.c_double),
                ("halo_exchanges", ctypes.c_int64), ("halo_ms", ctypes.c_double)]


@dataclass
class Params:
    """msa_params (include/msa.h); real quantities in the paper's Omega = [0,1]^2 units."""
    batch: int
    height: int
    width: int
    channels: int
    alpha: float = 1.0
    beta: float = 1.0
    radius: int = 2
    kernel: int = KERNEL_WENDLAND
    eps_x: float = 0.0
    eps_c: float = 57.0
    dt: float = 0.25
    rho: float = 1.0
    gamma: float = 1.0
    kappa: float = 1.0
    tau: float = 0.0
    sigma: float = 0.0
    theta: float = 1.0
    iters_per_round: int = 1
    rounds: int = 1
    shard: int = SHARD_NONE
    rank: int = 0
    world: int = 1
    device: int = 0
    nccl_id: bytes | None = field(default=None, repr=False)
    scheme: int = SCHEME_CP_ROUNDS

    @staticmethod
    def from_solver(B: int, H: int, W: int, C: int, sp: dict, **kw) -> "Params":
        keys = ("alpha", "beta", "radius", "kernel", "eps_x", "eps_c", "dt", "rho", "gamma", "kappa", "tau",
                "sigma", "theta", "iters_per_round", "rounds")
        if "scheme" in sp and "scheme" not in kw:
            kw = dict(kw, scheme=sp["scheme"])
        return Params(batch=B, height=H, width=W, channels=C, **{k: sp[k] for k in keys}, **kw)

    def c(self) -> tuple[_CParams, object]:
        d = asdict(self)
        nid = d.pop("nccl_id")
        keep = None
        ptr = None
        if nid is not None:
            keep = ctypes.create_string_buffer(bytes(nid), 128)
            ptr = ctypes.cast(keep, ctypes.c_void_p)
        return _CParams(**d, nccl_id=ptr), keep


_lib = None


def build(force: bool = False, verbose: bool = False) -> str:
    from . import _build
    return _build.build(force=force, verbose=verbose)


def lib():
    """The loaded libmsa.so. Raises if it has not been built (no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run paper_2510_16154_b200.build() (nvcc, sm_100a)")
        L = ctypes.CDLL(LIB_PATH)
        P, V, I32, I64, SZ = ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        PI32, PI64, PSZ, PD = (ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64),
                               ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_double))
        PP = ctypes.POINTER(_CParams)
        sig = {
            "msa_abi_version": ([], ctypes.c_int),
            "msa_last_error": ([], ctypes.c_char_p),
            "msa_workspace_bytes": ([PP, PSZ], ctypes.c_int),
            "msa_partition_rows": ([I32, I32, I32, I32, PI32, PI32, PI32], ctypes.c_int),
            "msa_nccl_unique_id": ([V], ctypes.c_int),
            "msa_halo_plan": ([I32, I32, I32, I32, I32, V, I32, PI32], ctypes.c_int),
            "msa_init": ([PP, V, ctypes.c_int, V, SZ, V, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
            "msa_reset": ([P, V, ctypes.c_int], ctypes.c_int),
            "msa_step": ([P, I32], ctypes.c_int),
            "msa_solve": ([P, V], ctypes.c_int),
            "msa_solve_until": ([P, ctypes.c_double, ctypes.c_double, I32, V, PI32, PI32], ctypes.c_int),
            "msa_solve_until_balanced": ([P, ctypes.c_double, ctypes.c_double, I32, ctypes.c_double, ctypes.c_double,
                                          V, V, PI32, PI32], ctypes.c_int),
            "msa_labels": ([P, ctypes.c_float, V, V, V, I32, ctypes.c_int], ctypes.c_int),
            "msa_label_margin": ([P, ctypes.c_float, V], ctypes.c_int),
            "msa_get_field": ([P, I32, V, ctypes.c_int, PI32, PI32], ctypes.c_int),
            "msa_set_field": ([P, I32, V, ctypes.c_int], ctypes.c_int),
            "msa_get_stats": ([P, V, I32, PI32], ctypes.c_int),
            "msa_state_bytes": ([P, PSZ], ctypes.c_int),
            "msa_get_state": ([P, V, SZ], ctypes.c_int),
            "msa_set_state": ([P, V, SZ], ctypes.c_int),
            "msa_query": ([P, ctypes.POINTER(Info)], ctypes.c_int),
            "msa_set_timing": ([P, ctypes.c_int], ctypes.c_int),
            "msa_get_timing": ([P, PD, PI64, PD, PI64], ctypes.c_int),
            "msa_sync": ([P], ctypes.c_int),
            "msa_dal": ([P, ctypes.POINTER(_DalParams), P, P, P, P, P, P], ctypes.c_int),
            "msa_dal_gradient": ([P, ctypes.POINTER(_DalParams), P, P, P, P, P], ctypes.c_int),
            "msa_dal_admm": ([P, ctypes.POINTER(_DalParams), P, P, P, I32, P, P, P], ctypes.c_int),
            "msa_free": ([P], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != MSA_OK:
        raise MsaError(rc, lib().msa_last_error().decode(errors="replace"))


def workspace_bytes(p: Params) -> int:
    cp, _keep = p.c()
    n = ctypes.c_size_t(0)
    _check(lib().msa_workspace_bytes(ctypes.byref(cp), ctypes.byref(n)))
    return n.value


def partition_rows(height: int, world: int, rank: int, radius: int) -> tuple[int, int, int]:
    r0, nr, g = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    _check(lib().msa_partition_rows(height, world, rank, radius, ctypes.byref(r0), ctypes.byref(nr), ctypes.byref(g)))
    return r0.value, nr.value, g.value


HALO_ITER, HALO_ROUND, HALO_MU = 0, 1, 2


class HaloOp(ctypes.Structure):
    _fields_ = [("field", ctypes.c_int32), ("peer", ctypes.c_int32), ("send", ctypes.c_int32),
                ("row0", ctypes.c_int32), ("nrows", ctypes.c_int32)]


def halo_plan(height: int, world: int, rank: int, radius: int, phase: int) -> list[tuple]:
    """msa_halo_plan: [(field, peer, send, row0, nrows)] - host only, no GPU needed."""
    n = ctypes.c_int32(0)
    _check(lib().msa_halo_plan(height, world, rank, radius, phase, None, 0, ctypes.byref(n)))
    buf = (HaloOp * max(n.value, 1))()
    _check(lib().msa_halo_plan(height, world, rank, radius, phase, buf, n.value, ctypes.byref(n)))
    return [(o.field, o.peer, o.send, o.row0, o.nrows) for o in buf[:n.value]]


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().msa_nccl_unique_id(buf))
    return buf.raw


def _torch():
    import torch
    return torch


def _ptr_of(x, n: int | None = None, what: str = "buffer", out: bool = False, dtype=np.float32,
            device: int | None = None):
    """(pointer, on_device, keepalive) of a numpy array or a torch tensor of n elements of dtype.
    Inputs are converted (numpy) or made contiguous (torch); outputs must already be contiguous
    and of the right dtype, since the library writes into them. Sizes are checked: the library
    trusts them. A CUDA tensor must live on the context's device (params.device): the library's
    kernels and copies run there."""
    if isinstance(x, np.ndarray):
        if out:
            if x.dtype != dtype or not x.flags.c_contiguous or not x.flags.writeable:
                raise TypeError(f"{what}: need a writeable C-contiguous {np.dtype(dtype).name} array")
        else:
            x = np.ascontiguousarray(x, dtype=dtype)
        if n is not None and x.size != n:
            raise ValueError(f"{what}: expected {n} elements, got {x.size} (shape {x.shape})")
        return x.ctypes.data, 0, x
    torch = _torch()
    if isinstance(x, torch.Tensor):
        tdt = {np.float32: torch.float32, np.int32: torch.int32}[dtype]
        if x.dtype != tdt:
            raise TypeError(f"{what}: need a {tdt} tensor, got {x.dtype}")
        if not x.is_contiguous():
            if out:
                raise TypeError(f"{what}: output tensor must be contiguous")
            x = x.contiguous()
        if n is not None and x.numel() != n:
            raise ValueError(f"{what}: expected {n} elements, got {x.numel()} (shape {tuple(x.shape)})")
        if x.is_cuda and device is not None and x.device.index != device:
            raise ValueError(f"{what}: tensor is on cuda:{x.device.index}, the context runs on cuda:{device}")
        return x.data_ptr(), int(x.is_cuda), x
    raise TypeError(f"{what}: unsupported buffer type {type(x)}")


class Solver:
    """One msa context (include/msa.h msa_init .. msa_free)."""

    def __init__(self, params: Params, image, stream=None, torch_workspace: bool = True):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("msa needs a CUDA device (sm_100a); there is no CPU path")
        self.params = params
        L = lib()
        cp, self._keep_id = params.c()
        self._cparams = cp
        nbytes = workspace_bytes(params)
        self._ws = None
        ws_ptr = None
        dev = torch.device("cuda", params.device)
        if torch_workspace:
            self._ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
            base = self._ws.data_ptr()
            ws_ptr = (base + 255) // 256 * 256
        if stream is None:
            stream = torch.cuda.current_stream(dev)
        self._stream = stream
        sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream or 0)
        ptr, on_dev, keep = _ptr_of(image, params.batch * params.height * params.width * params.channels, "image",
                                     device=params.device)
        ctx = ctypes.c_void_p()
        _check(L.msa_init(ctypes.byref(cp), ptr, on_dev, ws_ptr, nbytes, sptr or None, ctypes.byref(ctx)))
        self._ctx = ctx

    # -- lifecycle
    def close(self) -> None:
        if getattr(self, "_ctx", None):
            lib().msa_free(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- hot path
    def reset(self, image) -> None:
        p = self.params
        ptr, on_dev, keep = _ptr_of(image, p.batch * p.height * p.width * p.channels, "image", device=p.device)
        _check(lib().msa_reset(self._ctx, ptr, on_dev))
        if not on_dev:
            self.sync()

    def step(self, n_iters: int) -> None:
        _check(lib().msa_step(self._ctx, int(n_iters)))

    def solve(self) -> list[dict]:
        n = max(self.params.rounds, 1)
        buf = (RoundStats * n)()
        _check(lib().msa_solve(self._ctx, buf))
        return [buf[r].as_dict(self.params.channels) for r in range(self.params.rounds)]

    def solve_until(self, tol_residual: float = 0.0, tol_gap: float = 0.0, max_rounds: int = 100):
        """Rounds until al_residual <= tol_residual or |gap| <= tol_gap (Alg. 2's stop criterion);
        returns (records, converged)."""
        buf = (RoundStats * max(max_rounds, 1))()
        n, conv = ctypes.c_int32(0), ctypes.c_int32(0)
        _check(lib().msa_solve_until(self._ctx, float(tol_residual), float(tol_gap), int(max_rounds), buf,
                                     ctypes.byref(n), ctypes.byref(conv)))
        return [buf[r].as_dict(self.params.channels) for r in range(n.value)], bool(conv.value)

    def solve_until_balanced(self, max_rounds: int, tol_residual: float = 0.0, tol_gap: float = 0.0,
                             rb_mu: float = 10.0, rb_tau: float = 2.0):
        """Multiplier rounds with the residual-balancing penalty (msa_solve_until_balanced):
        returns (records, dual_residuals, converged)."""
        buf = (RoundStats * max(max_rounds, 1))()
        dres = np.zeros(max(max_rounds, 1))
        rr, conv = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().msa_solve_until_balanced(self._ctx, float(tol_residual), float(tol_gap), int(max_rounds),
                                              float(rb_mu), float(rb_tau), buf, dres.ctypes.data, ctypes.byref(rr),
                                              ctypes.byref(conv)))
        n = rr.value
        return [buf[r].as_dict(self.params.channels) for r in range(n)], dres[:n], bool(conv.value)

    def labels(self, delta: float = 0.1, max_k: int = 0, out=None):
        """Returns (labels int32 [nb][rows][W], n_clusters int32 [nb], palette [nb][max_k][C] or None);
        rows = this rank's slab rows in rows mode, else H. Cluster ids and palettes are global."""
        info = self.query()
        nb, H, W, C = info.nimages, info.nrows, self.params.width, self.params.channels
        if out is None:
            lab = np.empty((nb, H, W), dtype=np.int32)
            cnt = np.empty(nb, dtype=np.int32)
            pal = np.zeros((nb, max_k, C), dtype=np.float32) if max_k > 0 else None
            _check(lib().msa_labels(self._ctx, ctypes.c_float(delta), lab.ctypes.data, cnt.ctypes.data,
                                    pal.ctypes.data if pal is not None else None, max_k, 0))
            return lab, cnt, pal
        lab, cnt, pal = out  # torch CUDA tensors
        for t, n, dt, what in ((lab, nb * H * W, np.int32, "labels"), (cnt, nb, np.int32, "n_clusters"),
                               (pal, nb * max_k * C, np.float32, "palette")):
            if t is None:
                continue
            ptr, on_dev, _ = _ptr_of(t, n, what, out=True, dtype=dt, device=self.params.device)
            if not on_dev:
                raise TypeError(f"{what}: out= takes CUDA tensors (device outputs)")
        if max_k > 0 and pal is None:
            raise ValueError("palette tensor needed when max_k > 0")
        _check(lib().msa_labels(self._ctx, ctypes.c_float(delta), lab.data_ptr(), cnt.data_ptr(),
                                pal.data_ptr() if pal is not None else None, max_k, 1))
        return lab, cnt, pal

    # -- fields and state
    def label_margin(self, delta: float = 0.1) -> np.ndarray:
        """Stage-(i) decision margin of Q(c; delta) per image (reading R17; msa_label_margin)."""
        out = np.zeros(self.query().nimages, dtype=np.float32)
        _check(lib().msa_label_margin(self._ctx, ctypes.c_float(delta), out.ctypes.data))
        return out

    def get_field(self, which: int = FIELD_C, out=None) -> np.ndarray:
        info = self.query()
        C = self.params.channels
        nm = 2 * C if which in (FIELD_P, FIELD_MU) else C
        if out is None:
            out = np.empty((info.nimages, info.nrows, self.params.width, nm), dtype=np.float32)
            _check(lib().msa_get_field(self._ctx, which, out.ctypes.data, 0, None, None))
            return out
        ptr, on_dev, keep = _ptr_of(out, info.nimages * info.nrows * self.params.width * nm, "out", out=True,
                                     device=self.params.device)
        _check(lib().msa_get_field(self._ctx, which, ptr, on_dev, None, None))
        return out

    def set_field(self, which: int, arr) -> None:
        info = self.query()
        C = self.params.channels
        nm = 2 * C if which in (FIELD_P, FIELD_MU) else C
        ptr, on_dev, keep = _ptr_of(arr, info.nimages * info.nrows * self.params.width * nm, "field",
                                     device=self.params.device)
        _check(lib().msa_set_field(self._ctx, which, ptr, on_dev))

    def stats(self) -> list[dict]:
        n = ctypes.c_int32(0)
        _check(lib().msa_get_stats(self._ctx, None, 0, ctypes.byref(n)))
        buf = (RoundStats * max(n.value, 1))()
        _check(lib().msa_get_stats(self._ctx, buf, n.value, ctypes.byref(n)))
        return [buf[r].as_dict(self.params.channels) for r in range(n.value)]

    def get_state(self) -> bytes:
        n = ctypes.c_size_t(0)
        _check(lib().msa_state_bytes(self._ctx, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().msa_get_state(self._ctx, buf, n.value))
        return buf.raw

    def set_state(self, blob: bytes) -> None:
        buf = ctypes.create_string_buffer(blob, len(blob))
        _check(lib().msa_set_state(self._ctx, buf, len(blob)))

    def query(self) -> Info:
        info = Info()
        _check(lib().msa_query(self._ctx, ctypes.byref(info)))
        return info

    def set_timing(self, enable: bool) -> None:
        _check(lib().msa_set_timing(self._ctx, int(enable)))

    def get_timing(self) -> dict:
        it, rd = ctypes.c_double(), ctypes.c_double()
        nit, nrd = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().msa_get_timing(self._ctx, ctypes.byref(it), ctypes.byref(nit), ctypes.byref(rd),
                                    ctypes.byref(nrd)))
        return dict(iter_ms=it.value, iter_launches=nit.value, round_ms=rd.value, round_launches=nrd.value)

    def sync(self) -> None:
        _check(lib().msa_sync(self._ctx))

    # -- NEXT-1: DAL control optimisation (Algorithm 1)
    def _vmu(self, v, mu):
        keep = []
        out = []
        n = self.params.height * self.params.width * 2 * self.params.channels
        for a, what in ((v, "v"), (mu, "mu")):
            if a is None:
                out.append(None)
            else:
                ptr, on_dev, k = _ptr_of(a, n, what, device=self.params.device)
                if on_dev:
                    raise TypeError(f"{what}: host array expected")
                keep.append(k)
                out.append(ptr)
        return out, keep

    def dal(self, d: "DalParams", eps, v=None, mu=None, return_stop: bool = False):
        """Optimises eps ([steps][2]) from the given guess; returns (eps, J_hist, sigma_hist[, stop]). With
        d.eta / d.eta_grad (Remark 3.4) the run may stop early: J_hist has run + 1 entries, sigma_hist run,
        stop = (iterations run, 0 cap | 1 cost stationarity | 2 projected gradient)."""
        e = np.ascontiguousarray(eps, dtype=np.float64).copy()
        assert e.shape == (d.steps, 2)
        Jh = np.zeros(d.iters + 1)
        sh = np.zeros(max(d.iters, 1))
        stop = np.zeros(2, dtype=np.int32)
        (vp, mp), keep = self._vmu(v, mu)
        _check(lib().msa_dal(self._ctx, ctypes.byref(d.c_struct()), e.ctypes.data, vp, mp, Jh.ctypes.data,
                             sh.ctypes.data, stop.ctypes.data))
        run = int(stop[0])
        out = (e, Jh[:run + 1], sh[:run])
        return out + ((run, int(stop[1])),) if return_stop else out

    def dal_admm(self, d: "DalParams", eps, outer: int, v=None, mu=None, return_gamma: bool = False):
        """Algorithm 2 with DAL as line 5 (d.cost must be 1): returns (eps, J_hist [outer][iters+1],
        records [outer][, gamma_hist [outer]]); the final mu is FIELD_MU. d.gamma_ls = 1 chooses each
        ascent step by the two-way Armijo search (the remark after Algorithm 2)."""
        e = np.ascontiguousarray(eps, dtype=np.float64).copy()
        assert e.shape == (d.steps, 2)
        Jh = np.zeros((max(outer, 1), d.iters + 1))
        gh = np.zeros(max(outer, 1))
        buf = (RoundStats * max(outer, 1))()
        (vp, mp), keep = self._vmu(v, mu)
        _check(lib().msa_dal_admm(self._ctx, ctypes.byref(d.c_struct()), e.ctypes.data, vp, mp, int(outer),
                                  Jh.ctypes.data, buf, gh.ctypes.data))
        out = (e, Jh[:outer], [buf[r].as_dict(self.params.channels) for r in range(outer)])
        return out + (gh[:outer],) if return_gamma else out

    def dal_gradient(self, d: "DalParams", eps, v=None, mu=None):
        e = np.ascontiguousarray(eps, dtype=np.float64)
        g = np.zeros_like(e)
        J = ctypes.c_double()
        (vp, mp), keep = self._vmu(v, mu)
        _check(lib().msa_dal_gradient(self._ctx, ctypes.byref(d.c_struct()), e.ctypes.data, vp, mp, ctypes.byref(J),
                                      g.ctypes.data))
        return J.value, g


def quantize(image, delta: float = 0.1, radius: int = 5, iters_per_round: int = 100, rounds: int = 10,
             max_k: int = 64, scheme: int = SCHEME_CP_ROUNDS, **params):
    """One call: evolve an image with the pixel multi-agent dynamics + TV control and label it by
    Q(c; delta). image: float32 [H][W][C] or [B][H][W][C] in [0, 1], row 0 = bottom (numpy or torch).
    Defaults are the BASELINE recipe in pixel units: alpha h = 8, rho/h = gamma/h =
    2.5, beta = 1, dt = 0.25, eps_c = 57, Wendland kernel, eps_x by
    reading R2; any msa_params field can be overridden by keyword (Omega units).
    Returns (c [B][H][W][C] float32, labels [B][H][W] int32, n_clusters [B] int32,
    palette [B][max_k][C] float32 or None)."""
    shape = tuple(image.shape)
    if len(shape) == 3:
        image = image[None]
    B, H, W, C = (int(v) for v in image.shape)
    h = 1.0 / (W - 1) if W > 1 else 1.0
    kw = dict(alpha=8.0 / h, beta=1.0, radius=radius, eps_c=57.0, dt=0.25, rho=2.5 * h, gamma=2.5 * h,
              iters_per_round=iters_per_round, rounds=rounds, scheme=scheme)
    kw.update(params)
    with Solver(Params(batch=B, height=H, width=W, channels=C, **kw), image) as s:
        s.solve()
        c = s.get_field(FIELD_C)
        lab, cnt, pal = s.labels(delta, max_k)
    if len(shape) == 3:
        return c[0], lab[0], cnt[:1], pal[:1] if pal is not None else None
    return c, lab, cnt, pal
