"""CPU oracle for the detector-tomography hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2404_02844_b200`` never imports it, and the two share no code.

This module is a ctypes shim around ``qdt_oracle.c`` (plain fp64 C, ``-O2
-ffp-contract=off``, OpenMP with a thread-count-independent deterministic split: results are
bit-identical for any ``set_threads(n)``): argument marshalling only, every number is
computed in C.
Each C function cites the PAPER.md passage it follows.

Parity status: every function below is pinned by a
``-m "not gpu"`` test in ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qdt_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=gnu11", "-fopenmp",
             "-shared", "-fPIC", _SRC, "-o", tmp, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, f64 = ctypes.c_int64, ctypes.c_double
        P64 = ctypes.POINTER(ctypes.c_int64)
        L.or_band.argtypes = [f64, i64, f64, i64, P64, P64]
        L.or_band.restype = None
        L.or_poisson_pmf.argtypes = [i64, f64]
        L.or_poisson_pmf.restype = f64
        L.or_build_probes.argtypes = [_f64p, i64, i64, f64, i64, _i64p, _i64p, _i64p,
                                      ctypes.c_void_p]
        L.or_build_probes.restype = ctypes.c_int
        L.or_project_simplex.argtypes = [_f64p, i64, _f64p, _f64p]
        L.or_project_simplex.restype = f64
        L.or_project_rows.argtypes = [_f64p, i64, i64, _f64p]
        L.or_project_rows.restype = None
        L.or_forward.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, _f64p, ctypes.c_void_p, i64,
                                 _f64p]
        L.or_forward.restype = None
        L.or_laplacian.argtypes = [_f64p, i64, i64, _f64p]
        L.or_laplacian.restype = None
        L.or_backward.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, _f64p, _f64p, i64, f64,
                                  _f64p]
        L.or_backward.restype = None
        L.or_regul.argtypes = [_f64p, i64, i64]
        L.or_regul.restype = f64
        L.or_objective.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, _f64p, _f64p, i64, f64]
        L.or_objective.restype = f64
        L.or_kkt.argtypes = [_f64p, _f64p, i64, i64, ctypes.POINTER(f64)]
        L.or_kkt.restype = f64
        L.or_sqs_weights.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, f64, _f64p]
        L.or_sqs_weights.restype = None
        L.or_power_iteration.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, i64]
        L.or_power_iteration.restype = f64
        L.or_solve.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, _f64p, i64, f64, f64, i64,
                               ctypes.c_int, ctypes.c_int, i64, ctypes.c_void_p, _f64p,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.POINTER(f64), ctypes.c_void_p, f64, ctypes.c_void_p,
                               ctypes.POINTER(f64)]
        L.or_solve.restype = i64
        L.or_smooth.argtypes = [_f64p, i64, i64, i64, i64, _f64p]
        L.or_smooth.restype = None
        L.or_hess_diag.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, f64, _f64p]
        L.or_hess_diag.restype = None
        L.or_row_argmax.argtypes = [_f64p, i64, i64, _i64p]
        L.or_row_argmax.restype = None
        L.or_newton_direction.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, _f64p, i64, f64, _f64p,
                                          ctypes.c_void_p, f64, i64, _f64p, ctypes.POINTER(f64)]
        L.or_newton_direction.restype = i64
        L.or_newton.argtypes = [_i64p, _i64p, _i64p, _f64p, i64, i64, _f64p, i64, f64, _f64p, i64, f64,
                                f64, i64, f64, i64, ctypes.c_int, _f64p, _f64p, _i64p, _i64p, _f64p,
                                ctypes.POINTER(i64)]
        L.or_newton.restype = i64
        L.or_set_threads.argtypes = [ctypes.c_int]
        L.or_set_threads.restype = None
        L.or_get_threads.argtypes = []
        L.or_get_threads.restype = ctypes.c_int
        L.or_newton_set_cg_rtol.argtypes = [f64]
        L.or_newton_set_cg_rtol.restype = None
        _lib = L
    return _lib


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Probes:
    """Banded F in probe-major storage (lo, len, off, val) as built by the oracle."""

    def __init__(self, alpha2, M: int, c_sigma: float = 6.0, margin: int = 16):
        alpha2 = _f(alpha2)
        D = alpha2.shape[0]
        self.D, self.M = D, int(M)
        self.alpha2 = alpha2
        self.lo = np.zeros(D, np.int64)
        self.len = np.zeros(D, np.int64)
        self.off = np.zeros(D + 1, np.int64)
        L = lib()
        rc = L.or_build_probes(alpha2, D, self.M, c_sigma, margin, self.lo, self.len, self.off,
                               None)
        if rc != 0:
            raise ValueError("or_build_probes: invalid arguments")
        self.nnz = int(self.off[-1])
        self.val = np.zeros(self.nnz, np.float64)
        L.or_build_probes(alpha2, D, self.M, c_sigma, margin, self.lo, self.len, self.off,
                          self.val.ctypes.data)

    @classmethod
    def from_banded(cls, lo, length, val, M: int):
        """A banded F given directly (the test hook qdt_probes_from_banded's counterpart)."""
        self = cls.__new__(cls)
        self.lo = np.ascontiguousarray(lo, dtype=np.int64)
        self.len = np.ascontiguousarray(length, dtype=np.int64)
        self.D, self.M = int(self.lo.shape[0]), int(M)
        self.alpha2 = None
        self.off = np.concatenate([[0], np.cumsum(self.len)]).astype(np.int64)
        self.nnz = int(self.off[-1])
        self.val = _f(val).copy()
        assert self.val.shape[0] == self.nnz
        return self

    @property
    def hi(self):
        return self.lo + self.len - 1

    def dense(self) -> np.ndarray:
        """Dense D x M copy of F (small instances only)."""
        F = np.zeros((self.D, self.M))
        for d in range(self.D):
            F[d, self.lo[d]:self.lo[d] + self.len[d]] = self.val[self.off[d]:self.off[d + 1]]
        return F

    def _args(self):
        return self.lo, self.len, self.off, self.val, self.D


def band(mu: float, M: int, c_sigma: float = 6.0, margin: int = 16):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    lib().or_band(float(mu), int(M), float(c_sigma), int(margin), ctypes.byref(lo),
                  ctypes.byref(hi))
    return lo.value, hi.value


def poisson_pmf(k: int, mu: float) -> float:
    return lib().or_poisson_pmf(int(k), float(mu))


def project_simplex(x):
    x = _f(x)
    y = np.empty_like(x)
    w = np.empty_like(x)
    tau = lib().or_project_simplex(x, x.shape[0], y, w)
    return y, tau


def project_rows(X):
    X = _f(X)
    Y = np.empty_like(X)
    lib().or_project_rows(X, X.shape[0], X.shape[1], Y)
    return Y


def forward(F: Probes, Theta, P=None):
    """R = F Theta - P (P omitted: R = F Theta)."""
    Theta = _f(Theta)
    N = Theta.shape[1] if Theta.ndim == 2 else 1
    R = np.empty((F.D, N))
    Pp = None if P is None else _f(P)
    lib().or_forward(*F._args(), Theta, None if Pp is None else Pp.ctypes.data, N, R)
    return R


def backward(F: Probes, R, Theta, gamma: float = 0.0):
    """G = F^T R + gamma L Theta (half gradient)."""
    R, Theta = _f(R), _f(Theta)
    N = Theta.shape[1]
    G = np.empty((F.M, N))
    lib().or_backward(*F._args(), F.M, R, Theta, N, float(gamma), G)
    return G


def laplacian(Theta):
    Theta = _f(Theta)
    LT = np.empty_like(Theta)
    lib().or_laplacian(Theta, Theta.shape[0], Theta.shape[1], LT)
    return LT


def regul(Theta) -> float:
    Theta = _f(Theta)
    return lib().or_regul(Theta, Theta.shape[0], Theta.shape[1])


def objective(F: Probes, P, Theta, gamma: float) -> float:
    P, Theta = _f(P), _f(Theta)
    return lib().or_objective(*F._args(), F.M, P, Theta, Theta.shape[1], float(gamma))


def kkt(Theta, G):
    Theta, G = _f(Theta), _f(G)
    rp = ctypes.c_double()
    r = lib().or_kkt(Theta, G, Theta.shape[0], Theta.shape[1], ctypes.byref(rp))
    return r, rp.value


def sqs_weights(F: Probes, gamma: float):
    w = np.empty(F.M)
    lib().or_sqs_weights(*F._args(), F.M, float(gamma), w)
    return w


def power_iteration(F: Probes, k_pow: int = 100) -> float:
    return lib().or_power_iteration(*F._args(), F.M, int(k_pow))


STEP_SQS, STEP_LIPSCHITZ, STEP_BB, STEP_BB_LS = 0, 1, 2, 3


def solve(F: Probes, P, gamma: float, tol: float, iters: int, step: int = STEP_SQS,
          accel: int = 0, kkt_every: int = 1, theta0=None, theta_prev=None, fista_t: float = 0.0):
    """Projected-gradient solve; returns dict(theta, trace, kkt, kkt_paper, iters_done, step,
    theta_prev, fista_t).  FISTA resume: theta_prev = Theta_{k-1}, fista_t = tau_k."""
    P = _f(P)
    N = P.shape[1]
    Theta = np.empty((F.M, N))
    Tprev = np.empty((F.M, N))
    trace = np.full(iters + 1, np.nan)
    kt = np.full(iters + 1, np.nan)
    kp = np.full(iters + 1, np.nan)
    st = ctypes.c_double()
    tau = ctypes.c_double()
    t0 = None if theta0 is None else _f(theta0)
    tp = None if theta_prev is None else _f(theta_prev)
    done = lib().or_solve(*F._args(), F.M, P, N, float(gamma), float(tol), int(iters), int(step),
                          int(accel), int(kkt_every), None if t0 is None else t0.ctypes.data,
                          Theta, trace.ctypes.data, kt.ctypes.data, kp.ctypes.data,
                          ctypes.byref(st), None if tp is None else tp.ctypes.data, float(fista_t),
                          Tprev.ctypes.data, ctypes.byref(tau))
    return dict(theta=Theta, trace=trace[:done + 1], kkt=kt[:done + 1], kkt_paper=kp[:done + 1],
                iters_done=int(done), step=st.value, theta_prev=Tprev, fista_t=tau.value)


def set_threads(n: int = 0):
    """Thread count of the oracle (0: all cores).  Results do not depend on it."""
    lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(lib().or_get_threads())


def smooth(Theta, exclude: int = 100, div: int = 50):
    """Long-range smoothing of PAPER.md:307-314 (reading R13)."""
    Theta = _f(Theta)
    out = np.empty_like(Theta)
    lib().or_smooth(Theta, Theta.shape[0], Theta.shape[1], int(exclude), int(div), out)
    return out


def hess_diag(F: Probes, gamma: float):
    """h_i = 2 (sum_d F_{d,i}^2 + gamma L_ii): Hessian diagonal per Fock row (Table 1)."""
    h = np.empty(F.M)
    lib().or_hess_diag(F.lo, F.len, F.off, F.val, F.D, F.M, float(gamma), h)
    return h


def row_argmax(Theta):
    Theta = _f(Theta)
    m = np.empty(Theta.shape[0], dtype=np.int64)
    lib().or_row_argmax(Theta, Theta.shape[0], Theta.shape[1], m)
    return m


NEWTON_DEFAULTS = dict(eps_active=1e-8, cg_max=50, switch_tol=1e-4, max_ls=60)


def newton_direction(F: Probes, P, gamma: float, Theta, m=None, eps_active: float = 1e-8,
                     cg_max: int = 50, cg_rtol: float = -1.0):
    """One two-metric Newton direction (stage 1: m None; stage 2: row maxima m).
    cg_rtol >= 0 replaces CG's forcing term (pins).  Returns (p, slope, cg_iterations)."""
    P, Theta = _f(P), _f(Theta)
    lib().or_newton_set_cg_rtol(float(cg_rtol))
    p = np.empty_like(Theta)
    sl = ctypes.c_double()
    mp = None if m is None else np.ascontiguousarray(m, dtype=np.int64)
    it = lib().or_newton_direction(F.lo, F.len, F.off, F.val, F.D, F.M, P, P.shape[1], float(gamma),
                                   Theta, None if mp is None else mp.ctypes.data, float(eps_active),
                                   int(cg_max), p, ctypes.byref(sl))
    return p, sl.value, int(it)


def newton(F: Probes, P, gamma: float, max_iter: int, eps_kkt: float = 0.0, theta0=None,
           eps_active: float = 1e-8, cg_max: int = 50, switch_tol: float = 1e-4, max_ls: int = 60,
           armijo: int = 0):
    """Two-stage two-metric projected truncated Newton (reading R16).
    armijo 0: the paper's printed line-search test; 1: the secant form."""
    P = _f(P)
    N = P.shape[1]
    Theta = np.full((F.M, N), 1.0 / N) if theta0 is None else _f(theta0).copy()
    tr = np.full(max_iter + 1, np.nan)
    kk = np.full(max_iter + 1, np.nan)
    st = np.zeros(max_iter + 1, dtype=np.int64)
    cg = np.zeros(max_iter + 1, dtype=np.int64)
    al = np.full(max_iter + 1, np.nan)
    sw = ctypes.c_int64()
    lib().or_newton_set_cg_rtol(-1.0)
    k = lib().or_newton(F.lo, F.len, F.off, F.val, F.D, F.M, P, N, float(gamma), Theta, int(max_iter),
                        float(eps_kkt), float(eps_active), int(cg_max), float(switch_tol), int(max_ls),
                        int(armijo), tr, kk, st, cg, al, ctypes.byref(sw))
    return dict(theta=Theta, trace=tr[:k + 1], kkt=kk[:k + 1], stage=st[:k], cg=cg[:k], alpha=al[:k],
                iters_done=int(k), switch=int(sw.value))

