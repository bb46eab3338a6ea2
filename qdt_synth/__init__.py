"""Seeded synthetic workloads for the detector-tomography hot path.

This module is shared by the tests (oracle and CUDA sides) and by ``bench.py``.  It holds
none of the method's arithmetic: it only draws the inputs ``alpha2`` (probe means
|alpha_d|^2) and ``P`` (D x N outcome probabilities).  To synthesise ``P`` it needs a
forward model ``P = F Theta_true`` (eq. Matrix); it uses its OWN
coherent-state matrix from ``scipy.stats.poisson`` on a deliberately wider window
(+-8 sigma + 24) than the solver's band, so the data come from the (nearly) untruncated
physics, not from either implementation under test.

The five configurations are BASELINE.json ``configs`` (recipes: DESIGN.md "Input recipe");
the paper's own workloads (Zenodo experimental data; Liu et al.'s simulated
F/P) are not available, these stand in for them with the same shapes.
"""
from __future__ import annotations

import dataclasses
import warnings

import numpy as np
import scipy.sparse as sp
import scipy.special as sps
import scipy.stats as st


@dataclasses.dataclass
class Instance:
    name: str
    alpha2: np.ndarray          # (D,) sorted probe means |alpha_d|^2
    M: int                      # Fock cutoff
    P: np.ndarray               # (D, N) outcome probabilities
    gamma: float
    iters: int
    theta_true: object = None   # dense (M,N) ndarray or scipy.sparse CSR, when kept

    @property
    def D(self):
        return self.alpha2.shape[0]

    @property
    def N(self):
        return self.P.shape[1]


def coherent_matrix(alpha2: np.ndarray, M: int) -> sp.csr_matrix:
    """Generator-side F (D x M): Poisson pmf on a +-8 sigma + 24 window (scipy)."""
    rows, cols, vals = [], [], []
    for d, mu in enumerate(alpha2):
        s = np.sqrt(mu)
        lo = max(0, int(np.floor(mu - 8 * s - 24)))
        hi = min(M - 1, int(np.ceil(mu + 8 * s + 24)))
        k = np.arange(lo, hi + 1)
        v = st.poisson.pmf(k, mu) if mu > 0 else (k == 0).astype(float)
        rows.append(np.full(k.shape, d))
        cols.append(k)
        vals.append(v)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals)
    return sp.csr_matrix((v, (r, c)), shape=(alpha2.shape[0], M))


def _multinomial_rows(rng, E: np.ndarray, shots: int) -> np.ndarray:
    """Reading R6: one multinomial per probe over N+1 categories (N outcomes + 'above the
    cutoff' with probability 1 - sum_n E[d,n]); the extra category is dropped."""
    E = np.clip(E, 0.0, None)
    rest = np.clip(1.0 - E.sum(axis=1, keepdims=True), 0.0, None)
    pv = np.concatenate([E, rest], axis=1)
    pv /= pv.sum(axis=1, keepdims=True)
    out = np.empty_like(E)
    for d in range(E.shape[0]):                       # probe order d = 0..D-1
        out[d] = rng.multinomial(shots, pv[d])[:-1] / shots
    return out


def _binom_thin(k_max: int, eta: float) -> np.ndarray:
    """B[k, j] = Bin(j; k, eta) for k, j < k_max (dense; small cutoffs only)."""
    k = np.arange(k_max)[:, None]
    j = np.arange(k_max)[None, :]
    with np.errstate(all="ignore"):
        B = st.binom.pmf(j, k, eta)
    return np.nan_to_num(B)


# ---------------------------------------------------------------- ground-truth detectors
def theta_tiny(M: int = 50, bins: int = 9, eta: float = 0.8) -> np.ndarray:
    """9-bin spatially multiplexed click detector: j ~ Bin(k, eta) photons land uniformly in
    9 bins; outcome n = number of occupied bins (N = 10).  Occupancy by the exact DP
    O_{j+1}(n) = O_j(n) n/9 + O_j(n-1) (10-n)/9."""
    N = bins + 1
    O = np.zeros((M, N))
    O[0, 0] = 1.0
    for j in range(M - 1):
        for n in range(N):
            O[j + 1, n] = O[j, n] * n / bins + (O[j, n - 1] * (bins - (n - 1)) / bins if n else 0)
    return _binom_thin(M, eta) @ O


def theta_medium(M: int = 1000, N: int = 100, eta: float = 0.9) -> np.ndarray:
    """n' ~ Bin(k, 0.9); outcome n = min(n', N-1)."""
    B = _binom_thin(M, eta)
    T = np.zeros((M, N))
    T[:, :N - 1] = B[:, :N - 1]
    T[:, N - 1] = np.clip(1.0 - B[:, :N - 1].sum(axis=1), 0.0, None)
    return T


def theta_large(M: int = 10000, N: int = 1000, eta: float = 0.85, width: float = 10.0,
                jitter: float = 0.02) -> np.ndarray:
    """n' ~ Bin(k, 0.85); reading x ~ Normal(n', (0.02 n')^2) (x = 0 when n' = 0); N linear
    bins of width 10 photons over [0, 10^4), x < 10 -> bin 0, x >= 9990 -> bin N-1."""
    npr = np.arange(M)[:, None].astype(float)
    edges = width * np.arange(1, N)[None, :]           # interior edges 10, 20, ..., 9990
    sig = jitter * npr
    with np.errstate(all="ignore"):
        C = sps.ndtr((edges - npr) / np.where(sig > 0, sig, 1.0))   # P(x < edge)
    C[0, :] = 1.0                                      # n' = 0: x = 0 < every edge
    Gm = np.empty((M, N))
    Gm[:, 0] = C[:, 0]
    Gm[:, 1:N - 1] = np.diff(C, axis=1)
    Gm[:, N - 1] = 1.0 - C[:, -1]
    Gm = np.clip(Gm, 0.0, None)
    B = _binom_thin(M, eta)                            # k x n'
    return B @ Gm


def theta_logbins_sparse(M: int, N: int, eta: float = 0.9) -> sp.csr_matrix:
    """n' ~ Bin(k, eta); outcome n = min(N-1, floor(N ln(1+n') / ln(1+n'_max))) with
    n'_max = eta (M-1).  Row k = differences of the binomial CDF at the bin edges."""
    npmax = eta * (M - 1)
    Lg = np.log1p(npmax)
    nprime = np.arange(int(np.floor(npmax)) + 2)
    b = np.minimum(N - 1, np.floor(N * np.log1p(nprime) / Lg)).astype(np.int64)
    # first n' of every bin (bins may be empty)
    first = np.full(N + 1, nprime.shape[0], dtype=np.int64)
    ub, idx = np.unique(b, return_index=True)
    first[ub] = idx
    for n in range(N - 1, -1, -1):                     # empty bins: edge = next bin's edge
        first[n] = min(first[n], first[n + 1])
    first[N] = np.iinfo(np.int64).max // 4             # the last bin absorbs the tail
    k = np.arange(M, dtype=float)
    mean, sd = eta * k, np.sqrt(eta * (1 - eta) * k)
    lo_e, hi_e = mean - 12 * sd - 2, mean + 12 * sd + 2
    rows, cols, vals = [], [], []
    edge_f = first.astype(float)
    for n in range(N):
        a, c = edge_f[n], edge_f[n + 1]                # bin n = [a, c)
        sel = np.nonzero((c > lo_e) & (a <= hi_e + 1))[0]
        if sel.size == 0:
            continue
        kk = k[sel]
        with np.errstate(all="ignore"), warnings.catch_warnings():
            warnings.simplefilter("ignore", DeprecationWarning)   # integral values passed as float
            Fc = np.where(c - 1 >= kk, 1.0, sps.bdtr(np.minimum(c - 1, kk), kk, eta))
            Fa = np.where(a - 1 < 0, 0.0, np.where(a - 1 >= kk, 1.0,
                                                    sps.bdtr(np.maximum(a - 1, 0), kk, eta)))
        v = np.clip(Fc - Fa, 0.0, None)
        keep = v > 0
        rows.append(sel[keep])
        cols.append(np.full(keep.sum(), n))
        vals.append(v[keep])
    T = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(M, N))
    # renormalise rows against the CDF differencing roundoff
    s = np.asarray(T.sum(axis=1)).ravel()
    return sp.diags(1.0 / s) @ T


def theta_logbins_rows(M: int, N: int, eta: float = 0.9, chunk: int = 1 << 16) -> sp.csr_matrix:
    """The same Theta_true as theta_logbins_sparse, built row-major and vectorised over
    (row, bin) pairs (the per-bin loop is too slow at Stress: M = 10^6, N = 10^4)."""
    npmax = eta * (M - 1)
    Lg = np.log1p(npmax)
    nprime = np.arange(int(np.floor(npmax)) + 2)
    b = np.minimum(N - 1, np.floor(N * np.log1p(nprime) / Lg)).astype(np.int64)
    first = np.full(N + 1, nprime.shape[0], dtype=np.int64)
    ub, idx = np.unique(b, return_index=True)
    first[ub] = idx
    for n in range(N - 1, -1, -1):
        first[n] = min(first[n], first[n + 1])
    first[N] = np.iinfo(np.int64).max // 4
    edge_f = first.astype(float)
    rows_all, cols_all, vals_all = [], [], []
    for k0 in range(0, M, chunk):
        k = np.arange(k0, min(M, k0 + chunk), dtype=float)
        mean, sd = eta * k, np.sqrt(eta * (1 - eta) * k)
        lo_e, hi_e = mean - 12 * sd - 2, mean + 12 * sd + 2
        # bins n with c_n > lo_e and a_n <= hi_e + 1, c_n = edge_f[n + 1], a_n = edge_f[n]
        nlo = np.searchsorted(edge_f[1:], lo_e, side="right")          # first n with c_n > lo_e
        nhi = np.searchsorted(edge_f[:N], hi_e + 1, side="right")      # one past the last a_n <= hi_e + 1
        cnt = np.maximum(nhi - nlo, 0)
        # the CDF once per bin edge of each row (cnt + 1 edges), then differences of neighbours
        ce = np.where(cnt > 0, cnt + 1, 0)
        r = np.repeat(np.arange(k.shape[0]), ce)
        n = nlo[r] + (np.arange(ce.sum()) - np.repeat(np.cumsum(ce) - ce, ce))
        kk = k[r]
        e = edge_f[n]
        with np.errstate(all="ignore"), warnings.catch_warnings():
            warnings.simplefilter("ignore", DeprecationWarning)   # integral values passed as float
            Fe = np.where(e - 1 < 0, 0.0, np.where(e - 1 >= kk, 1.0, sps.bdtr(np.clip(e - 1, 0, kk), kk, eta)))
        last = np.zeros(r.shape[0], dtype=bool)
        if r.shape[0]:
            last[np.cumsum(ce)[ce > 0] - 1] = True
        lo_i = np.nonzero(~last)[0]
        v = np.clip(Fe[lo_i + 1] - Fe[lo_i], 0.0, None)
        keep = v > 0
        rows_all.append((r[lo_i] + k0)[keep])
        cols_all.append(n[lo_i][keep])
        vals_all.append(v[keep])
    T = sp.csr_matrix((np.concatenate(vals_all), (np.concatenate(rows_all), np.concatenate(cols_all))),
                      shape=(M, N))
    s = np.asarray(T.sum(axis=1)).ravel()
    return sp.diags(1.0 / s) @ T


# ---------------------------------------------------------------- the five configs
def tiny(seed: int = 0) -> Instance:
    M, D = 50, 100
    alpha2 = np.linspace(0.0, 40.0, D)
    T = theta_tiny(M)
    rng = np.random.Generator(np.random.PCG64(seed))
    E = coherent_matrix(alpha2, M) @ T
    P = _multinomial_rows(rng, E, 10 ** 5)
    return Instance("tiny", alpha2, M, P, 1e-3, 2000, T)


def medium(seed: int = 0) -> Instance:
    M, N, D = 1000, 100, 2000
    rng = np.random.Generator(np.random.PCG64(seed))
    alpha2 = np.sort(rng.uniform(0.0, 800.0, D))       # drawn before the noise
    T = theta_medium(M, N)
    E = coherent_matrix(alpha2, M) @ T
    P = _multinomial_rows(rng, E, 10 ** 6)
    return Instance("medium", alpha2, M, P, 1e-4, 2000, T)


def large(seed: int = 0) -> Instance:
    M, N, D = 10 ** 4, 1000, 2 * 10 ** 4
    alpha2 = np.geomspace(0.1, 8000.0, D)
    T = theta_large(M, N)
    E = np.asarray(coherent_matrix(alpha2, M) @ T)
    rng = np.random.Generator(np.random.PCG64(seed))
    P = rng.poisson(np.clip(E, 0, None) * 1e6) / 1e6   # independent Poisson per cell
    return Instance("large", alpha2, M, P, 1e-4, 200, T)


def megascale(seed: int = 0, keep_theta: bool = False) -> Instance:
    M, N, D = 10 ** 6, 100, 10 ** 4
    alpha2 = np.geomspace(1.0, 9e5, D)
    T = theta_logbins_sparse(M, N)
    E = np.asarray((coherent_matrix(alpha2, M) @ T).todense())
    rng = np.random.Generator(np.random.PCG64(seed))
    P = _multinomial_rows(rng, E, 10 ** 7)
    return Instance("megascale", alpha2, M, P, 1e-5, 100, T if keep_theta else None)


def stress_cut(seed: int = 0) -> Instance:
    """Stress-shaped cut-down: M = 10^5, N = 10^3, D = 2000 log-spaced probes,
    log bins, noiseless P = F Theta_true."""
    M, N, D = 10 ** 5, 1000, 2000
    alpha2 = np.geomspace(1.0, 0.9 * M * 0.9, D)
    T = theta_logbins_sparse(M, N)
    P = np.asarray((coherent_matrix(alpha2, M) @ T).todense())
    return Instance("stress_cut", alpha2, M, P, 1e-5, 3, T)


def stress(seed: int = 0, M: int = 10 ** 6, N: int = 10 ** 4, D: int = 2 * 10 ** 4,
           keep_theta: bool = False) -> Instance:
    """BASELINE Stress: M = 10^6, N = 10^4 (10^10 elements), D = 2 10^4 probes log-spaced in
    [1, 9 10^5], Theta_true = efficiency 0.9 thinning into 10^4 log bins, noiseless
    P = F Theta_true, gamma = 1e-5, 200 iterations.  Smaller M / N / D give the Stress-shaped
    parity instances (probe means up to 0.9 * 0.9 M, as stress_cut)."""
    mu_max = 9e5 if M == 10 ** 6 else 0.81 * M
    alpha2 = np.geomspace(1.0, mu_max, D)
    T = theta_logbins_rows(M, N)
    P = np.asarray((coherent_matrix(alpha2, M) @ T).todense())
    return Instance("stress" if M == 10 ** 6 else f"stress_M{M}_N{N}", alpha2, M, P, 1e-5, 200,
                    T if keep_theta else None)


def random_instance(seed: int, D: int, M: int, N: int, mu_max: float | None = None,
                    gamma: float = 1e-3) -> Instance:
    """Small random instance for parity sweeps: sorted uniform probe means, P rows drawn from
    a Dirichlet (not necessarily consistent with any Theta)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    mu_max = float(M) * 0.8 if mu_max is None else mu_max
    alpha2 = np.sort(rng.uniform(0.0, mu_max, D))
    P = rng.dirichlet(np.ones(N), size=D)
    return Instance(f"random{seed}", alpha2, M, P, gamma, 50, None)




# ---------------------------------------------------------------- the paper's own detector
TMD_R, TMD_ETA_LOOP, TMD_ETA_DET = 0.91644, 0.90524, 0.528   # fitted values


def tmd_click_probs(i: np.ndarray, bins: int = 150) -> np.ndarray:
    """Bin-click probabilities of the time-multiplexed detector for Fock inputs i (eq. pj_fock,
    PAPER.md:208-217): p_1 = 1 - (1 - R eta_det)^i, p_j = 1 - [1 - (1-R)^2 R^-1 (R eta_loop)^(j-1)
    eta_det]^i for j >= 2.  Returns (len(i), bins)."""
    R, el, ed = TMD_R, TMD_ETA_LOOP, TMD_ETA_DET
    j = np.arange(1, bins + 1, dtype=float)
    q = np.where(j == 1, R * ed, (1 - R) ** 2 / R * (R * el) ** (j - 1) * ed)   # per-photon probability
    i = np.asarray(i, dtype=float)[:, None]
    return -np.expm1(i * np.log1p(-q)[None, :])


def theta_tmd(M: int, bins: int = 150, block: int = 2048) -> np.ndarray:
    """Analytic POVM of the detector: outcome n = number of clicked bins among
    the first `bins` (N = bins + 1 = 151), the Poisson-binomial distribution of independent bin
    clicks with probabilities p_j(i); computed by the exact DP over bins (after j bins only
    counts <= j are reachable), blocks of rows on a thread pool (numpy releases the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor
    N = bins + 1
    T = np.empty((M, N))

    def run(r0):
        r1 = min(M, r0 + block)
        p = tmd_click_probs(np.arange(r0, r1), bins)
        q = 1.0 - p
        dp = np.zeros((r1 - r0, N))
        dp[:, 0] = 1.0
        for j in range(bins):
            pj, qj = p[:, j:j + 1], q[:, j:j + 1]
            hi = dp[:, :j + 1] * pj
            dp[:, :j + 1] *= qj
            dp[:, 1:j + 2] += hi
        T[r0:r1] = dp

    with ThreadPoolExecutor(min(16, os.cpu_count() or 1)) as ex:
        list(ex.map(run, range(0, M, block)))
    return T


def paper_tmd(D: int = 1076, seed: int = 0, trials: int = 5 * 10 ** 5, noiseless: bool = False,
              gamma: float = 1e-5, M: int | None = None) -> Instance:
    """Paper-shaped synthetic workload: quadratic probes |alpha_d|^2 = d^2
    (PAPER.md:112, 190), cutoff M covering the last probe's band, the analytic time-multiplexed
    detector POVM with the paper's fitted parameters, multinomial noise at 5e5 trials per probe
    (reading R6).  D = 1076 gives the paper's shape (M = 1 210 581, N = 151,
    PAPER.md:124) with its nearest-neighbour gamma = 1e-5."""
    alpha2 = np.arange(D, dtype=float) ** 2
    mu = alpha2[-1]
    if M is None and D == 1076:
        M = 1210581                  # the paper's cutoff at its D
    if M is None:                    # just past the last probe's band
        M = int(mu + 6 * np.sqrt(mu) + 100)
    else:                            # |alpha_d|^2 ~ d^2 scaled so the last band reaches M - 100
        mu_top = (-3.0 + np.sqrt(9.0 + M - 100)) ** 2
        alpha2 = alpha2 * (mu_top / max(mu, 1.0))
    T = theta_tmd(M)
    E = np.asarray(coherent_matrix(alpha2, M) @ T)
    if noiseless:
        P = E
    else:
        rng = np.random.Generator(np.random.PCG64(seed))
        P = _multinomial_rows(rng, E, trials)
    return Instance(f"paper_tmd{D}", alpha2, M, P, gamma, 300, T)


def fidelities(theta: np.ndarray, theta_true: np.ndarray) -> np.ndarray:
    """Per-outcome fidelity of diagonal POVM elements (eq. fidelities, diagonal
    form): F_n = (sum_i sqrt(theta_in t_in))^2 / (sum_i theta_in sum_i t_in)."""
    num = np.sum(np.sqrt(np.clip(theta, 0, None) * theta_true), axis=0) ** 2
    den = theta.sum(0) * theta_true.sum(0)
    return np.where(den > 0, num / np.where(den > 0, den, 1), np.nan)


CONFIGS = {"tiny": tiny, "medium": medium, "large": large, "megascale": megascale,
           "stress": stress, "stress_cut": stress_cut, "paper_tmd": paper_tmd}
