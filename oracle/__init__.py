"""ctypes wrapper of the fp64 CPU oracle (oracle/msa_oracle.c).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package. The product
package (paper_2510_16154_b200) never imports it and shares no code with it.

Parity status: every function here is pinned by tests/test_oracle_pins.py
 except the composite agent+TV trajectory, which has no
closed form and is pinned by invariants only: P8 (mean), P9
(constant fixed point), P21 (transpose / channel-permutation equivariance,
tests/test_oracle_symmetry.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import replace, dataclass, asdict

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmsa_oracle.so")
_lib = None

NSTAT_FIXED = 8
STAT_NAMES = ["E_TV", "E_fid", "P", "D", "gap", "residual", "rho", "nonfinite"]


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "msa_oracle.c")
    hdr = os.path.join(_HERE, "msa_oracle.h")
    newest = max(os.path.getmtime(src), os.path.getmtime(hdr))
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < newest:
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fopenmp", "-fPIC",
                               "-shared", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


class _Params(ctypes.Structure):
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32), ("channels", ctypes.c_int32),
                ("radius", ctypes.c_int32), ("kernel", ctypes.c_int32), ("iters_per_round", ctypes.c_int32),
                ("rounds", ctypes.c_int32), ("scheme", ctypes.c_int32)] + [
        (n, ctypes.c_double) for n in ("hx", "hy", "alpha", "beta", "eps_x", "eps_c", "dt", "rho", "gamma",
                                       "kappa", "tau", "sigma", "theta")]


@dataclass
class Params:
    height: int
    width: int
    channels: int
    radius: int = 2
    kernel: int = 0
    iters_per_round: int = 1
    rounds: int = 1
    hx: float = 0.0
    hy: float = 0.0
    alpha: float = 1.0
    beta: float = 1.0
    eps_x: float = 0.0
    eps_c: float = 57.0
    dt: float = 0.25
    rho: float = 1.0
    gamma: float = 1.0
    kappa: float = 1.0
    tau: float = 0.0
    sigma: float = 0.0
    theta: float = 1.0
    scheme: int = 0  # 0: CP iterations + multiplier rounds; 1: single-loop linearised ADMM (NEXT-2)

    def c(self) -> _Params:
        d = asdict(self)
        return _Params(**{k: d[k] for k in ("height", "width", "channels", "radius", "kernel", "iters_per_round",
                                            "rounds", "scheme")},
                       **{k: float(d[k]) for k in ("hx", "hy", "alpha", "beta", "eps_x", "eps_c", "dt", "rho",
                                                   "gamma", "kappa", "tau", "sigma", "theta")})

    @staticmethod
    def from_solver(H: int, W: int, C: int, sp: dict) -> "Params":
        return Params(height=H, width=W, channels=C, radius=sp["radius"], kernel=sp["kernel"],
                      iters_per_round=sp["iters_per_round"], rounds=sp["rounds"], alpha=sp["alpha"],
                      beta=sp["beta"], eps_x=sp["eps_x"], eps_c=sp["eps_c"], dt=sp["dt"], rho=sp["rho"],
                      gamma=sp["gamma"], kappa=sp["kappa"], tau=sp["tau"], sigma=sp["sigma"], theta=sp["theta"],
                      scheme=sp.get("scheme", 0))


_D = ctypes.c_void_p


class _DalParams(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int32), ("cost", ctypes.c_int32), ("iters", ctypes.c_int32),
                ("max_ls", ctypes.c_int32), ("sigma0", ctypes.c_double), ("b", ctypes.c_double),
                ("c", ctypes.c_double), ("ex_lo", ctypes.c_double), ("ex_hi", ctypes.c_double),
                ("ec_lo", ctypes.c_double), ("ec_hi", ctypes.c_double), ("rho", ctypes.c_double),
                ("eta", ctypes.c_double), ("eta_grad", ctypes.c_double)]


@dataclass
class DalParams:
    """NEXT-1 DAL settings (oracle/msa_oracle.h mo_dal_params)."""
    M: int
    cost: int = 0           # 0: J of eq:cost_functional, 1: L~ with fixed v, mu
    iters: int = 10
    max_ls: int = 30
    sigma0: float = 1.0
    b: float = 0.5
    c: float = 1e-4
    ex_lo: float = 2.0      # E = [2, 1100]^2
    ex_hi: float = 1100.0
    ec_lo: float = 2.0
    ec_hi: float = 1100.0
    rho: float = 1.0
    eta: float = 0.0        # Remark 3.4 cost stationarity tolerance (1e-10); 0: off
    eta_grad: float = 0.0   # Remark 3.4 projected-gradient tolerance; 0: off

    def c_struct(self) -> _DalParams:
        return _DalParams(**asdict(self))


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER(_Params)
        sig = {
            "mo_derive": ([P, P], ctypes.c_int),
            "mo_phi": ([ctypes.c_double, ctypes.c_int], ctypes.c_double),
            "mo_pair_r": ([ctypes.c_double] * 5, ctypes.c_double),
            "mo_window_size": ([ctypes.c_int], ctypes.c_int),
            "mo_grad": ([_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double], None),
            "mo_div": ([_D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double], None),
            "mo_agent_rhs": ([P, _D, _D], None),
            "mo_init_state": ([P, _D, _D, _D, _D, _D], None),
            "mo_iteration": ([P, ctypes.c_double, _D, _D, _D, _D, _D], None),
            "mo_round_stats": ([P, ctypes.c_double, _D, _D, _D, _D, _D], None),
            "mo_round_update": ([P, ctypes.c_double, _D, _D], None),
            "mo_iteration_lin": ([P, ctypes.c_double, _D, _D, _D], None),
            "mo_round_stats_lin": ([P, ctypes.c_double, _D, _D, _D, _D], None),
            "mo_run": ([P, _D, _D, _D, _D, _D, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double), _D,
                        ctypes.c_int32], ctypes.c_int),
            "mo_energy_K": ([P, _D, _D], ctypes.c_double),
            "mo_energy_L": ([P, ctypes.c_double, _D, _D, _D, _D], ctypes.c_double),
            "mo_energy_Ltilde": ([P, ctypes.c_double, _D, _D, _D, _D], ctypes.c_double),
            "mo_shrink_field": ([P, ctypes.c_double, _D, _D, _D], None),
            "mo_phi_prime": ([ctypes.c_double, ctypes.c_int], ctypes.c_double),
            "mo_agent_rhs_eps": ([P, ctypes.c_double, ctypes.c_double, _D, _D], None),
            "mo_agent_jtvp": ([P, ctypes.c_double, ctypes.c_double, _D, _D, _D], None),
            "mo_agent_deps": ([P, ctypes.c_double, ctypes.c_double, _D, _D, _D], None),
            "mo_dal_cost": ([P, ctypes.POINTER(_DalParams), _D, _D, _D, _D, _D], ctypes.c_double),
            "mo_dal_gradient": ([P, ctypes.POINTER(_DalParams), _D, _D, _D, _D, _D], ctypes.c_double),
            "mo_dal": ([P, ctypes.POINTER(_DalParams), _D, _D, _D, _D, _D, _D, _D], ctypes.c_int),
            "mo_labels": ([_D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_float, _D,
                           ctypes.POINTER(ctypes.c_int32), _D, ctypes.c_int32], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data


def derive(p: Params) -> Params:
    out = _Params()
    if _load().mo_derive(ctypes.byref(p.c()), ctypes.byref(out)) != 0:
        raise ValueError(f"invalid oracle params {p}")
    d = {f[0]: getattr(out, f[0]) for f in _Params._fields_}
    return Params(**d)


def phi(r: float, kernel: int = 0) -> float:
    return _load().mo_phi(r, kernel)


def pair_r(dx: float, dy: float, dc2: float, eps_x: float, eps_c: float) -> float:
    return _load().mo_pair_r(dx, dy, dc2, eps_x, eps_c)


def window_size(R: int) -> int:
    return _load().mo_window_size(R)


def grad(u: np.ndarray, hx: float, hy: float) -> np.ndarray:
    u = _f64(u)
    H, W, C = u.shape
    g = np.empty((H, W, 2 * C))
    _load().mo_grad(_ptr(u), _ptr(g), H, W, C, hx, hy)
    return g


def div(p: np.ndarray, hx: float, hy: float) -> np.ndarray:
    p = _f64(p)
    H, W, C2 = p.shape
    d = np.empty((H, W, C2 // 2))
    _load().mo_div(_ptr(p), _ptr(d), H, W, C2 // 2, hx, hy)
    return d


def agent_rhs(p: Params, c: np.ndarray) -> np.ndarray:
    c = _f64(c)
    assert c.shape == (p.height, p.width, p.channels), "field shape must match the params"
    F = np.empty_like(c)
    _load().mo_agent_rhs(ctypes.byref(derive(p).c()), _ptr(c), _ptr(F))
    return F


class State:
    """Oracle state of one image: c, cbar [H][W][C]; p, mu [H][W][2C]; rho; global iteration."""

    def __init__(self, p: Params, I: np.ndarray):
        self.params = p
        self.I = _f64(I)
        H, W, C = self.I.shape
        assert (H, W, C) == (p.height, p.width, p.channels)
        self.c = np.empty_like(self.I)
        self.cbar = np.empty_like(self.I)
        self.p = np.empty((H, W, 2 * C))
        self.mu = np.empty((H, W, 2 * C))
        _load().mo_init_state(ctypes.byref(p.c()), _ptr(self.I), _ptr(self.c), _ptr(self.cbar), _ptr(self.p),
                              _ptr(self.mu))
        self.rho = float(p.rho)
        self.iter = 0
        self.stats: list[np.ndarray] = []

    def run(self, n_iters: int) -> list[np.ndarray]:
        C = self.params.channels
        cap = n_iters // max(self.params.iters_per_round, 1) + 2
        st = np.zeros((cap, NSTAT_FIXED + C))
        rho = ctypes.c_double(self.rho)
        nr = _load().mo_run(ctypes.byref(self.params.c()), _ptr(self.I), _ptr(self.c), _ptr(self.cbar),
                            _ptr(self.p), _ptr(self.mu), self.iter, n_iters, ctypes.byref(rho), _ptr(st), cap)
        if nr < 0:
            raise ValueError("oracle rejected params")
        self.rho = rho.value
        self.iter += n_iters
        new = [st[r].copy() for r in range(nr)]
        self.stats.extend(new)
        return new

    def iteration(self) -> None:
        """One iteration (steps 1-3) without any round logic."""
        _load().mo_iteration(ctypes.byref(derive(self.params).c()), self.rho, _ptr(self.I), _ptr(self.c),
                             _ptr(self.cbar), _ptr(self.p), _ptr(self.mu))

    def round_stats(self) -> np.ndarray:
        C = self.params.channels
        st = np.zeros(NSTAT_FIXED + C)
        _load().mo_round_stats(ctypes.byref(derive(self.params).c()), self.rho, _ptr(self.I), _ptr(self.c),
                               _ptr(self.p), _ptr(self.mu), _ptr(st))
        return st

    def round_update(self) -> None:
        _load().mo_round_update(ctypes.byref(derive(self.params).c()), self.rho, _ptr(self.c), _ptr(self.mu))


def solve(p: Params, I: np.ndarray) -> State:
    """rounds x K iterations from the initial state (SURVEY.md §8(c) oracle block)."""
    s = State(p, I)
    s.run(p.rounds * p.iters_per_round)
    return s


def energy_K(p: Params, u, I) -> float:
    u, I = _f64(u), _f64(I)
    return _load().mo_energy_K(ctypes.byref(p.c()), _ptr(u), _ptr(I))


def energy_L(p: Params, rho: float, u, v, mu, I) -> float:
    u, v, mu, I = _f64(u), _f64(v), _f64(mu), _f64(I)
    return _load().mo_energy_L(ctypes.byref(p.c()), rho, _ptr(u), _ptr(v), _ptr(mu), _ptr(I))


def energy_Ltilde(p: Params, rho: float, u, v, mu, I) -> float:
    u, v, mu, I = _f64(u), _f64(v), _f64(mu), _f64(I)
    return _load().mo_energy_Ltilde(ctypes.byref(p.c()), rho, _ptr(u), _ptr(v), _ptr(mu), _ptr(I))


def shrink_field(p: Params, rho: float, c, mu) -> np.ndarray:
    c, mu = _f64(c), _f64(mu)
    v = np.empty_like(mu)
    _load().mo_shrink_field(ctypes.byref(derive(p).c()), rho, _ptr(c), _ptr(mu), _ptr(v))
    return v


def labels(c: np.ndarray, delta: float = 0.1, max_k: int = 0):
    """Q(c; delta) of reading R16 on a float32 [H][W][C] field -> (labels int32 [H][W], count, palette)."""
    c = np.ascontiguousarray(c, dtype=np.float32)
    H, W, C = c.shape
    lab = np.empty((H, W), dtype=np.int32)
    n = ctypes.c_int32(0)
    pal = np.zeros((max(max_k, 1), C), dtype=np.float32)
    rc = _load().mo_labels(_ptr(c), H, W, C, ctypes.c_float(delta), _ptr(lab), ctypes.byref(n), _ptr(pal), max_k)
    if rc != 0:
        raise ValueError("labels: non-finite or out-of-range field")
    return lab, n.value, pal[:min(max_k, n.value)] if max_k > 0 else None


def solve_until_balanced(p: Params, I, max_rounds: int, tol_residual: float = 0.0, tol_gap: float = 0.0,
                         rb_mu: float = 10.0, rb_tau: float = 2.0):
    """Multiplier rounds with residual-balancing penalty (SURVEY §8(f) NEXT-2 "adaptive rho"; the
    standard ADMM rule of Boyd et al., not in the paper, which fixes rho = gamma at PAPER.md:470).
    Round r runs K iterations and its multiplier update exactly as State.run (Alg. 2 lines 6-7, then
    rho <- kappa rho). With v^(r) = S_{beta/rho_r}(grad c^(r) - mu^(r)/rho_r) (the round's shrink, pre-update
    mu, reading R11), the primal residual is the record's ||v^(r) - grad c^(r)||_w and the dual residual
    s^(r) = rho_r ||div(v^(r) - v^(r-1))||_w (constraint v - grad u = 0: A = -grad, A^T = div, reading R6).
    From round 1 on: if r > rb_mu s then rho <- rb_tau rho, elif s > rb_mu r then rho <- rho / rb_tau (for
    the next round). The run stops after a round whose residual <= tol_residual or |gap| <= tol_gap
    (each test off at 0; reading R13), or after max_rounds. Returns (state, records, dual_residuals)."""
    st = State(p, _f64(I))
    q = derive(p)
    w = q.hx * q.hy
    K = p.iters_per_round
    recs, duals, v_prev = [], [], None
    for _ in range(max_rounds):
        mu_pre, rho_r = st.mu.copy(), st.rho
        rec = st.run(K)[-1]
        v = shrink_field(p, rho_r, st.c, mu_pre)
        s_dual = float("nan") if v_prev is None else rho_r * float(np.sqrt(w * np.sum(div(v - v_prev, q.hx, q.hy) ** 2)))
        recs.append(rec)
        duals.append(s_dual)
        v_prev = v
        if (tol_residual > 0 and rec[5] <= tol_residual) or (tol_gap > 0 and abs(rec[4]) <= tol_gap):
            break
        r_prim = rec[5]
        if s_dual == s_dual:  # from the second round on
            if r_prim > rb_mu * s_dual:
                st.rho *= rb_tau
            elif s_dual > rb_mu * r_prim:
                st.rho /= rb_tau
    return st, recs, duals


# ---------------------------------------------------------------- NEXT-1: DAL (Algorithm 1)
def phi_prime(r: float, kernel: int = 0) -> float:
    return _load().mo_phi_prime(r, kernel)


def agent_rhs_eps(p: Params, eps_x: float, eps_c: float, c) -> np.ndarray:
    c = _f64(c)
    F = np.empty_like(c)
    _load().mo_agent_rhs_eps(ctypes.byref(derive(p).c()), eps_x, eps_c, _ptr(c), _ptr(F))
    return F


def agent_jtvp(p: Params, eps_x: float, eps_c: float, c, lam) -> np.ndarray:
    c, lam = _f64(c), _f64(lam)
    g = np.empty_like(c)
    _load().mo_agent_jtvp(ctypes.byref(derive(p).c()), eps_x, eps_c, _ptr(c), _ptr(lam), _ptr(g))
    return g


def agent_deps(p: Params, eps_x: float, eps_c: float, c, lam) -> np.ndarray:
    c, lam = _f64(c), _f64(lam)
    out = np.zeros(2)
    _load().mo_agent_deps(ctypes.byref(derive(p).c()), eps_x, eps_c, _ptr(c), _ptr(lam), _ptr(out))
    return out


def _vmu(p: Params, v, mu):
    shape = (p.height, p.width, 2 * p.channels)
    v = _f64(np.zeros(shape) if v is None else v)
    mu = _f64(np.zeros(shape) if mu is None else mu)
    return v, mu


def dal_cost(p: Params, d: DalParams, eps, I, v=None, mu=None, return_state: bool = False):
    eps, I = _f64(eps), _f64(I)
    v, mu = _vmu(p, v, mu)
    cT = np.empty_like(I)
    J = _load().mo_dal_cost(ctypes.byref(p.c()), ctypes.byref(d.c_struct()), _ptr(eps), _ptr(I), _ptr(v), _ptr(mu),
                            _ptr(cT))
    return (J, cT) if return_state else J


def dual_value(p: Params, rho: float, c, mu, I) -> float:
    """Phi(mu) = min_v L(c, v, mu) at a fixed state c: the augmented Lagrangian of eq:complete_square
    at v = S_{beta/rho}(grad c - mu/rho) (eq:soft_threshold is the exact minimiser over v; pins P12/P13)."""
    v = shrink_field(p, rho, c, mu)
    return energy_L(p, rho, c, v, mu, I)


def dal_admm(p: Params, d: DalParams, eps, I, outer: int, v=None, mu=None, gamma_search: bool = False):
    """Algorithm 2 with Algorithm 1 as its line 5, step by step: for j = 0 ..
    outer-1: eps^(j) by dal() with the augmented-Lagrangian terminal at (v^(j-1), mu^(j)) (d.cost = 1),
    c^(j) = c(T; eps^(j)) by dal_cost(); v^(j) = S_{beta/rho}(grad c^(j) - mu^(j)/rho) (line 6,
    eq:soft_threshold); mu^(j+1) = mu^(j) + gamma^(j) (v^(j) - grad c^(j)) (line 7). v^(-1), mu^(0): the
    arguments or 0.

    gamma^(j): the fixed gamma, or (gamma_search) the two-way Armijo search of Algorithm 1 used for the
    ascent step as the remark after Algorithm 2 proposes: with g = v^(j) - grad c^(j)
    and Phi(mu') = min_v L(c(mu'), v, mu'), c(mu') the line-5 solution at (v^(j), mu') from eps^(j),
    a step t passes when Phi(mu^(j) + t g) >= Phi(mu^(j)) + c t |g|_w^2 (Phi(mu^(j)) at c^(j)); starting
    from gamma (then from the last accepted step) t grows by 1/b while it passes (the last passing t is
    kept) or shrinks by b until it passes, at most max_ls tests; none passes: no ascent step.
    Returns (eps, J_hist [outer][iters+1], c^(outer-1), v, mu[, gamma_hist])."""
    q = derive(p)
    d = replace(d, rho=q.rho)  # one penalty: the AL terminal of line 5 and the updates of lines 6-7
    eps = _f64(eps).copy()
    I = _f64(I)
    H, W, C = I.shape
    w = q.hx * q.hy
    v = np.zeros((H, W, 2 * C)) if v is None else _f64(v).copy()
    mu = np.zeros((H, W, 2 * C)) if mu is None else _f64(mu).copy()
    Jh, gh, c, gam = [], [], I.copy(), q.gamma
    for _ in range(outer):
        eps, J, _ = dal(p, d, eps, I, v, mu)
        Jh.append(np.concatenate([J, np.full(d.iters + 1 - len(J), J[-1])]))  # an early stop repeats its cost
        _, c = dal_cost(p, d, eps, I, v, mu, return_state=True)
        v = shrink_field(p, q.rho, c, mu)
        g = v - grad(c, q.hx, q.hy)
        step = q.gamma
        if gamma_search:
            phi0 = energy_L(p, q.rho, c, v, mu, I)
            g2 = w * float(np.sum(g * g))

            def passes(t):
                mt = mu + t * g
                et, _, _ = dal(p, d, eps, I, v, mt)
                _, ct = dal_cost(p, d, et, I, v, mt, return_state=True)
                return dual_value(p, q.rho, ct, mt, I) >= phi0 + d.c * t * g2

            tau, acc, evals = gam, -1.0, 1
            if passes(tau):
                acc = tau
                while evals < d.max_ls:
                    evals += 1
                    if not passes(tau / d.b):
                        break
                    tau /= d.b
                    acc = tau
            else:
                while evals < d.max_ls:
                    evals += 1
                    tau *= d.b
                    if passes(tau):
                        acc = tau
                        break
            step = acc if acc > 0 else 0.0
            gam = acc if acc > 0 else tau
        gh.append(step)
        mu = mu + step * g
    out = (eps, np.array(Jh), c, v, mu)
    return out + (np.array(gh),) if gamma_search else out


def dal_gradient(p: Params, d: DalParams, eps, I, v=None, mu=None):
    eps, I = _f64(eps), _f64(I)
    v, mu = _vmu(p, v, mu)
    g = np.empty_like(eps)
    J = _load().mo_dal_gradient(ctypes.byref(p.c()), ctypes.byref(d.c_struct()), _ptr(eps), _ptr(I), _ptr(v),
                                _ptr(mu), _ptr(g))
    return J, g


def dal(p: Params, d: DalParams, eps, I, v=None, mu=None, return_stop: bool = False):
    """Algorithm 1 from eps ([M][2], updated copy returned) -> (eps, J_hist, sigma_hist[, stop]).
    With the Remark 3.4 rules (d.eta, d.eta_grad) the run may end early: J_hist then has run + 1
    entries and sigma_hist run; stop = (iterations run, 0 cap | 1 cost stationarity | 2 gradient)."""
    eps = _f64(eps).copy()
    I = _f64(I)
    v, mu = _vmu(p, v, mu)
    Jh = np.zeros(d.iters + 1)
    sh = np.zeros(max(d.iters, 1))
    stop = np.zeros(2, dtype=np.int32)
    _load().mo_dal(ctypes.byref(p.c()), ctypes.byref(d.c_struct()), _ptr(eps), _ptr(I), _ptr(v), _ptr(mu), _ptr(Jh),
                   _ptr(sh), _ptr(stop))
    run = int(stop[0])
    out = (eps, Jh[:run + 1], sh[:run])
    return out + ((run, int(stop[1])),) if return_stop else out
