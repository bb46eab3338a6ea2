"""B200-native phase-insensitive quantum detector tomography (arXiv:2404.02844 hot path).

Thin Python binding over the C ABI in ``include/qdt.h`` (``libqdt.so``, built in-tree for
sm_100a).  The functions below carry the C names and only marshal arguments: numpy arrays
are passed as host pointers, CUDA torch tensors as device pointers (``mem_device = 1``).
Every step of the solve runs in the library's CUDA kernels; there is no CPU fallback -- if
``libqdt.so`` is missing or no GPU is present the calls raise.

    ctx = qdt_init(device=0)
    F = qdt_build_probes(ctx, alpha2, M)
    out = qdt_solve(ctx, F, P, gamma=1e-5, tol=0.0, iters=100)   # dict(theta, trace, kkt, info)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("QDT_LIB") or os.path.join(_HERE, "libqdt.so")   # QDT_LIB: in-tree A/B build

QDT_STEP_SQS, QDT_STEP_LIPSCHITZ, QDT_STEP_BB, QDT_STEP_BB_LS = 0, 1, 2, 3
STATUS = {0: "QDT_OK", 1: "QDT_ERR_INVALID_ARG", 2: "QDT_ERR_UNSORTED", 3: "QDT_ERR_NONFINITE",
          4: "QDT_ERR_OOM", 5: "QDT_ERR_CUDA", 6: "QDT_ERR_NCCL", 7: "QDT_ERR_TRUNCATED",
          8: "QDT_ERR_STATE"}

# every symbol include/qdt.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = ["qdt_init", "qdt_finalize", "qdt_last_error", "qdt_build_probes", "qdt_probes_free",
               "qdt_probes_export", "qdt_solve", "qdt_objective", "qdt_residual", "qdt_gradient",
               "qdt_step", "qdt_project_rows", "qdt_step_setup", "qdt_profile_enable",
               "qdt_profile_get", "qdt_launch_count", "qdt_nccl_unique_id", "qdt_shard_cuts",
               "qdt_smooth", "qdt_solve_newton", "qdt_probes_from_banded"]


class QdtError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


QDT_COMM_NCCL, QDT_COMM_INPROC = 0, 1


class InitOpts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p),
                ("comm", ctypes.c_int32), ("group_key", ctypes.c_int64)]


class ProbeOpts(ctypes.Structure):
    _fields_ = [("c_sigma", ctypes.c_double), ("margin", ctypes.c_int32),
                ("strict_mass", ctypes.c_int32)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("step", ctypes.c_int32), ("accel", ctypes.c_int32), ("theta0", ctypes.c_void_p),
                ("check_every", ctypes.c_int32), ("kkt_every", ctypes.c_int32),
                ("mem_device", ctypes.c_int32), ("gather_theta", ctypes.c_int32),
                ("use_graph", ctypes.c_int32), ("theta_prev", ctypes.c_void_p),
                ("fista_t", ctypes.c_double), ("theta_prev_out", ctypes.c_void_p),
                ("exchange", ctypes.c_int32)]


class NewtonOpts(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("cg_max", ctypes.c_int32), ("max_ls", ctypes.c_int32),
                ("mem_device", ctypes.c_int32), ("eps_active", ctypes.c_double),
                ("switch_tol", ctypes.c_double), ("theta0", ctypes.c_void_p), ("armijo", ctypes.c_int32)]


class NewtonInfo(ctypes.Structure):
    _fields_ = [("iters_done", ctypes.c_int64), ("switch_iter", ctypes.c_int64), ("cg_total", ctypes.c_int64),
                ("f_final", ctypes.c_double), ("kkt", ctypes.c_double), ("loop_ms", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SolveInfo(ctypes.Structure):
    _fields_ = [("iters_done", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("kkt0", ctypes.c_double), ("kkt", ctypes.c_double), ("kkt_paper", ctypes.c_double),
                ("f_final", ctypes.c_double), ("step_scalar", ctypes.c_double),
                ("k_begin", ctypes.c_int64), ("k_end", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("min_row_mass", ctypes.c_double), ("uncovered_rows", ctypes.c_int64),
                ("loop_ms", ctypes.c_double), ("fista_t", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libqdt.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    L.qdt_init.argtypes = [P(vp), P(InitOpts)]
    L.qdt_finalize.argtypes = [vp]
    L.qdt_last_error.argtypes = [vp]
    L.qdt_last_error.restype = ctypes.c_char_p
    L.qdt_build_probes.argtypes = [vp, vp, i64, i64, P(ProbeOpts), P(vp)]
    L.qdt_probes_free.argtypes = [vp]
    L.qdt_probes_from_banded.argtypes = [vp, i64, i64, vp, vp, vp, P(vp)]
    L.qdt_probes_export.argtypes = [vp, vp, P(i64), P(i64), P(i64), vp, vp, vp]
    L.qdt_solve.argtypes = [vp, vp, vp, i64, f64, f64, i64, P(SolveOpts), vp, vp, vp, P(SolveInfo)]
    L.qdt_objective.argtypes = [vp, vp, vp, vp, i64, f64, i32, P(f64), P(f64)]
    L.qdt_residual.argtypes = [vp, vp, vp, vp, i64, vp]
    L.qdt_gradient.argtypes = [vp, vp, vp, vp, i64, f64, vp]
    L.qdt_step.argtypes = [vp, vp, vp, vp, i64, f64, i32, vp]
    L.qdt_project_rows.argtypes = [vp, vp, i64, i64, vp]
    L.qdt_step_setup.argtypes = [vp, vp, f64, i32, vp, P(f64)]
    L.qdt_profile_enable.argtypes = [vp, i32]
    L.qdt_profile_get.argtypes = [vp, ctypes.c_char_p, P(i64), P(f64)]
    L.qdt_launch_count.argtypes = [vp, P(i64)]
    L.qdt_nccl_unique_id.argtypes = [vp]
    L.qdt_shard_cuts.argtypes = [vp, vp, i64, i64, i32, vp]
    L.qdt_smooth.argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
    L.qdt_solve_newton.argtypes = [vp, vp, vp, i64, f64, f64, P(NewtonOpts), vp, vp, vp, vp, vp, vp,
                                   P(NewtonInfo)]
    for s in ABI_SYMBOLS:
        if s != "qdt_last_error":
            getattr(L, s).restype = ctypes.c_int
    _lib = L
    return L


def _check(ctx, status):
    if status != 0:
        msg = load_library().qdt_last_error(ctx.ptr if isinstance(ctx, Context) else ctx)
        raise QdtError(status, (msg or b"").decode())


class Context:
    def __init__(self, ptr, device=0):
        self.ptr = ptr
        self.device = device

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.qdt_finalize(self.ptr)
            self.ptr = None


class Probes:
    def __init__(self, ctx, ptr, D, M):
        self.ctx, self.ptr, self.D, self.M = ctx, ptr, D, M

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.qdt_probes_free(self.ptr)
            self.ptr = None


def _host(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def _is_cuda_tensor(x):
    return hasattr(x, "is_cuda") and x.is_cuda


def _dev_arg(ctx: Context, x, name: str, shape=None):
    """A CUDA tensor argument: float64, contiguous, on ctx's device, of the given shape (the
    library reads raw fp64 memory).  Raises instead of converting silently."""
    import torch
    if not _is_cuda_tensor(x):
        raise TypeError(f"{name}: expected a CUDA tensor (P is one)")
    if x.dtype != torch.float64:
        raise TypeError(f"{name}: dtype {x.dtype}, the library computes in float64")
    if x.device.index != ctx.device:
        raise ValueError(f"{name}: on {x.device}, the context is on cuda:{ctx.device}")
    if shape is not None and tuple(x.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(x.shape)}, expected {tuple(shape)}")
    if not x.is_contiguous():
        raise ValueError(f"{name}: not contiguous")
    return x


def _order_after_torch(ctx: Context):
    """Device pointers are read on the library's own stream: finish the work torch queued on
    its current stream (the producer of P / theta0) before the call."""
    import torch
    torch.cuda.current_stream(ctx.device).synchronize()


def qdt_init(device: int = 0, rank: int = 0, nranks: int = 1, nccl_unique_id: bytes | None = None,
             cuda_stream: int | None = None, comm: int = QDT_COMM_NCCL, group_key: int = 0) -> Context:
    """comm = QDT_COMM_INPROC: virtual ranks of one process (each rank calls every collective
    function from its own thread; ctypes releases the GIL during the call)."""
    L = load_library()
    uid = ctypes.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id else None
    o = InitOpts(device, rank, nranks, ctypes.cast(uid, ctypes.c_void_p) if uid else None,
                 cuda_stream, int(comm), int(group_key))
    p = ctypes.c_void_p()
    st = L.qdt_init(ctypes.byref(p), ctypes.byref(o))
    if st != 0:
        raise QdtError(st, (L.qdt_last_error(None) or b"").decode())
    return Context(p, device)


def qdt_finalize(ctx: Context):
    if ctx.ptr:
        _check(ctx, load_library().qdt_finalize(ctx.ptr))
        ctx.ptr = None


def qdt_build_probes(ctx: Context, alpha2, M: int, c_sigma: float = 6.0, margin: int = 16,
                     strict_mass: bool = False) -> Probes:
    a = _host(alpha2)
    o = ProbeOpts(c_sigma, margin, int(strict_mass))
    p = ctypes.c_void_p()
    _check(ctx, load_library().qdt_build_probes(ctx.ptr, a.ctypes.data, a.shape[0], int(M),
                                                ctypes.byref(o), ctypes.byref(p)))
    return Probes(ctx, p, a.shape[0], int(M))


def qdt_probes_from_banded(ctx: Context, lo, length, vals, M: int) -> Probes:
    """Test hook: a probe handle from an arbitrary banded F (include/qdt.h)."""
    lo_, ln_ = _host(lo, np.int64), _host(length, np.int64)
    v = _host(vals)
    p = ctypes.c_void_p()
    _check(ctx, load_library().qdt_probes_from_banded(ctx.ptr, lo_.shape[0], int(M), lo_.ctypes.data,
                                                      ln_.ctypes.data, v.ctypes.data, ctypes.byref(p)))
    return Probes(ctx, p, lo_.shape[0], int(M))


def qdt_probes_export(ctx: Context, F: Probes, values: bool = True):
    L = load_library()
    nnz, kb, ke = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(ctx, L.qdt_probes_export(ctx.ptr, F.ptr, ctypes.byref(nnz), ctypes.byref(kb),
                                    ctypes.byref(ke), None, None, None))
    lo = np.zeros(F.D, np.int64)
    ln = np.zeros(F.D, np.int64)
    val = np.zeros(max(1, nnz.value), np.float64)
    _check(ctx, L.qdt_probes_export(ctx.ptr, F.ptr, None, None, None, lo.ctypes.data,
                                    ln.ctypes.data, val.ctypes.data if values else None))
    return dict(lo=lo, len=ln, val=val[:nnz.value], nnz=nnz.value, k_begin=kb.value,
                k_end=ke.value)


def qdt_solve(ctx: Context, F: Probes, P, gamma: float, tol: float = 0.0, iters: int = 100,
              step: int = QDT_STEP_SQS, accel: bool = False, theta0=None, check_every: int = 16,
              kkt_every: int = 1, gather_theta: bool = False, use_graph: bool = True,
              theta_out=None, theta_prev=None, fista_t: float = 0.0, want_prev: bool = False,
              no_theta: bool = False, exchange: int = 0, rows=None):
    """Projected-gradient solve.  P: numpy (host) or CUDA tensor (device, then theta0 and
    theta_out are device tensors too).  FISTA resume: theta_prev = Theta_{k-1}, fista_t = tau_k;
    want_prev returns Theta_{k-1} of the result as 'theta_prev'; no_theta copies no result out
    (theta None); rows: rows of theta_out (nranks > 1 without gather_theta: this rank's slice);
    exchange 1: band-aware residual exchange between ranks.  Returns dict(theta, trace, kkt, info[, theta_prev])."""
    L = load_library()
    dev = _is_cuda_tensor(P)
    prev_out = None
    if dev:
        import torch
        D, N = P.shape
        _dev_arg(ctx, P, "P", (F.D, N))
        rows = F.M if rows is None else int(rows)
        if theta_out is None and not no_theta:
            theta_out = torch.empty((rows, N), dtype=torch.float64, device=P.device)
        if theta_out is not None:
            _dev_arg(ctx, theta_out, "theta_out", (theta_out.shape[0], N))
        t0 = _dev_arg(ctx, theta0, "theta0", (rows, N)) if theta0 is not None else None
        tp = _dev_arg(ctx, theta_prev, "theta_prev", (rows, N)) if theta_prev is not None else None
        if want_prev:
            prev_out = torch.empty((rows, N), dtype=torch.float64, device=P.device)
        p_ptr, out_ptr = P.data_ptr(), (theta_out.data_ptr() if theta_out is not None else None)
        t0_ptr = t0.data_ptr() if t0 is not None else None
        tp_ptr = tp.data_ptr() if tp is not None else None
        po_ptr = prev_out.data_ptr() if prev_out is not None else None
        _order_after_torch(ctx)
    else:
        Pp = _host(P)
        D, N = Pp.shape
        if theta_out is None and not no_theta:
            theta_out = np.empty((F.M if rows is None else int(rows), N))
        t0 = _host(theta0) if theta0 is not None else None
        tp = _host(theta_prev) if theta_prev is not None else None
        if want_prev:
            prev_out = np.empty((F.M, N))
        p_ptr, out_ptr = Pp.ctypes.data, (theta_out.ctypes.data if theta_out is not None else None)
        t0_ptr = t0.ctypes.data if t0 is not None else None
        tp_ptr = tp.ctypes.data if tp is not None else None
        po_ptr = prev_out.ctypes.data if prev_out is not None else None
    trace = np.full(iters + 1, np.nan)
    kkt = np.full(iters + 1, np.nan)
    o = SolveOpts(step, int(accel), t0_ptr, check_every, kkt_every, int(dev), int(gather_theta),
                  int(use_graph), tp_ptr, float(fista_t), po_ptr, int(exchange))
    info = SolveInfo()
    _check(ctx, L.qdt_solve(ctx.ptr, F.ptr, p_ptr, N, float(gamma), float(tol), int(iters),
                            ctypes.byref(o), out_ptr, trace.ctypes.data, kkt.ctypes.data,
                            ctypes.byref(info)))
    k = info.iters_done
    out = dict(theta=theta_out, trace=trace[:k + 1], kkt=kkt[:k + 1], info=info.as_dict())
    if want_prev:
        out["theta_prev"] = prev_out
    return out


def qdt_objective(ctx: Context, F: Probes, P, theta, gamma: float):
    L = load_library()
    dev = _is_cuda_tensor(P)
    if dev:
        N = P.shape[1]
        Pp = _dev_arg(ctx, P, "P", (F.D, N))
        Tp = _dev_arg(ctx, theta, "theta", (F.M, N))
        pp, tp = Pp.data_ptr(), Tp.data_ptr()
        _order_after_torch(ctx)
    else:
        Pp, Tp = _host(P), _host(theta)
        pp, tp, N = Pp.ctypes.data, Tp.ctypes.data, Pp.shape[1]
    f, r = ctypes.c_double(), ctypes.c_double()
    _check(ctx, L.qdt_objective(ctx.ptr, F.ptr, pp, tp, N, float(gamma), int(dev), ctypes.byref(f),
                                ctypes.byref(r)))
    return f.value, r.value


def qdt_residual(ctx: Context, F: Probes, theta, P=None):
    Th = _host(theta)
    N = Th.shape[1]
    Pp = _host(P) if P is not None else None
    R = np.empty((F.D, N))
    _check(ctx, load_library().qdt_residual(ctx.ptr, F.ptr, Th.ctypes.data,
                                            Pp.ctypes.data if Pp is not None else None, N,
                                            R.ctypes.data))
    return R


def qdt_gradient(ctx: Context, F: Probes, R, theta, gamma: float):
    Rr, Th = _host(R), _host(theta)
    N = Th.shape[1]
    G = np.empty((F.M, N))
    _check(ctx, load_library().qdt_gradient(ctx.ptr, F.ptr, Rr.ctypes.data, Th.ctypes.data, N,
                                            float(gamma), G.ctypes.data))
    return G


def qdt_step(ctx: Context, F: Probes, P, theta, gamma: float, step: int = QDT_STEP_SQS):
    Pp, Th = _host(P), _host(theta)
    out = np.empty_like(Th)
    _check(ctx, load_library().qdt_step(ctx.ptr, F.ptr, Pp.ctypes.data, Th.ctypes.data,
                                        Th.shape[1], float(gamma), int(step), out.ctypes.data))
    return out


def qdt_project_rows(ctx: Context, X):
    Xx = _host(X)
    Y = np.empty_like(Xx)
    _check(ctx, load_library().qdt_project_rows(ctx.ptr, Xx.ctypes.data, Xx.shape[0],
                                                Xx.shape[1], Y.ctypes.data))
    return Y


def qdt_step_setup(ctx: Context, F: Probes, gamma: float, k_pow: int = 100, weights: bool = True,
                   power: bool = True):
    w = np.empty(F.M) if weights else None
    rho = ctypes.c_double()
    _check(ctx, load_library().qdt_step_setup(ctx.ptr, F.ptr, float(gamma), int(k_pow),
                                              w.ctypes.data if weights else None,
                                              ctypes.byref(rho) if power else None))
    return w, (rho.value if power else None)


def qdt_profile_enable(ctx: Context, enable: bool = True):
    _check(ctx, load_library().qdt_profile_enable(ctx.ptr, int(enable)))


def qdt_profile_get(ctx: Context, kernel: str):
    c, ms = ctypes.c_int64(), ctypes.c_double()
    _check(ctx, load_library().qdt_profile_get(ctx.ptr, kernel.encode(), ctypes.byref(c),
                                               ctypes.byref(ms)))
    return c.value, ms.value


def qdt_launch_count(ctx: Context) -> int:
    c = ctypes.c_int64()
    _check(ctx, load_library().qdt_launch_count(ctx.ptr, ctypes.byref(c)))
    return c.value


def qdt_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = load_library().qdt_nccl_unique_id(buf)
    if st != 0:
        raise QdtError(st, (load_library().qdt_last_error(None) or b"").decode())
    return buf.raw


def qdt_shard_cuts(lo, hi, M: int, nranks: int):
    lo_, hi_ = _host(lo, np.int64), _host(hi, np.int64)
    cuts = np.zeros(nranks + 1, np.int64)
    st = load_library().qdt_shard_cuts(lo_.ctypes.data, hi_.ctypes.data, lo_.shape[0], int(M),
                                       int(nranks), cuts.ctypes.data)
    if st != 0:
        raise QdtError(st, (load_library().qdt_last_error(None) or b"").decode())
    return cuts


def qdt_smooth(ctx: Context, theta, exclude: int = 100, div: int = 50, out=None):
    """Long-range smoothing: numpy in -> numpy out, CUDA tensor -> tensor."""
    L = load_library()
    if _is_cuda_tensor(theta):
        import torch
        th = _dev_arg(ctx, theta, "theta")
        out = torch.empty_like(th) if out is None else _dev_arg(ctx, out, "out", tuple(th.shape))
        _order_after_torch(ctx)
        _check(ctx, L.qdt_smooth(ctx.ptr, th.data_ptr(), th.shape[0], th.shape[1], int(exclude),
                                 int(div), 1, out.data_ptr()))
        return out
    th = _host(theta)
    out = np.empty_like(th) if out is None else out
    _check(ctx, L.qdt_smooth(ctx.ptr, th.ctypes.data, th.shape[0], th.shape[1], int(exclude),
                             int(div), 0, out.ctypes.data))
    return out


def qdt_solve_newton(ctx: Context, F: Probes, P, gamma: float, eps_kkt: float = 0.0, max_iter: int = 100,
                     cg_max: int = 50, max_ls: int = 60, eps_active: float = 1e-8, switch_tol: float = 1e-4,
                     theta0=None, armijo: int = 0):
    """Two-stage two-metric projected truncated Newton (include/qdt.h qdt_solve_newton; reading R16).
    Host numpy P / theta0 (single rank).  Returns dict(theta, trace, kkt, stage, cg, alpha, info)."""
    L = load_library()
    P = _host(P)
    D, N = P.shape
    M = F.M
    t0 = _host(theta0) if theta0 is not None else None
    o = NewtonOpts(int(max_iter), int(cg_max), int(max_ls), 0, float(eps_active), float(switch_tol),
                   t0.ctypes.data if t0 is not None else None, int(armijo))
    theta = np.empty((M, N))
    tr = np.full(max_iter + 1, np.nan)
    kk = np.full(max_iter + 1, np.nan)
    st = np.zeros(max(1, max_iter), dtype=np.int32)
    cg = np.zeros(max(1, max_iter), dtype=np.int32)
    al = np.full(max(1, max_iter), np.nan)
    info = NewtonInfo()
    _check(ctx, L.qdt_solve_newton(ctx.ptr, F.ptr, P.ctypes.data, N, float(gamma), float(eps_kkt),
                                   ctypes.byref(o), theta.ctypes.data, tr.ctypes.data, kk.ctypes.data,
                                   st.ctypes.data, cg.ctypes.data, al.ctypes.data, ctypes.byref(info)))
    k = int(info.iters_done)
    return dict(theta=theta, trace=tr[:k + 1], kkt=kk[:k + 1], stage=st[:k], cg=cg[:k], alpha=al[:k],
                info=info.as_dict())

