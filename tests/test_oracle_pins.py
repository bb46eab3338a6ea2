"""Pins for the CPU oracle (-m "not gpu").

Every check here ties oracle/ to something other than itself: closed forms, values the
paper's definitions fix, brute force on tiny inputs, high-precision evaluation (mpmath),
dense linear algebra (numpy), invariants.  Each test names the PAPER.md passage (or
DESIGN.md reading) it pins.  A plausible mistake anywhere in oracle/ (a dropped term, a
wrong sign or index, a transposed operand) fails at least one of them.
"""
import itertools
import math

import mpmath
import numpy as np
import pytest

import oracle
import qdt_synth as qs

mpmath.mp.dps = 40


# ----------------------------------------------------------------------------- P1, P2, P3
def _mp_pois(k, mu):
    """Poisson pmf at 40 digits: mu^k e^-mu / k! (eq. Fmatrix)."""
    mu = mpmath.mpf(mu)
    return mpmath.e ** (k * mpmath.log(mu) - mu - mpmath.loggamma(k + 1))


def test_poisson_closed_form_mu1():
    # F_{d,i} = |a|^{2i} e^{-|a|^2}/i! at |a|^2 = 1: (e^-1, e^-1, e^-1/2)
    e1 = math.exp(-1.0)
    assert oracle.poisson_pmf(0, 1.0) == pytest.approx(e1, rel=1e-15)
    assert oracle.poisson_pmf(1, 1.0) == pytest.approx(e1, rel=1e-15)
    assert oracle.poisson_pmf(2, 1.0) == pytest.approx(e1 / 2, rel=1e-15)
    # vacuum probe: F_{d,0} = 1, F_{d,i>0} = 0
    assert oracle.poisson_pmf(0, 0.0) == 1.0 and oracle.poisson_pmf(3, 0.0) == 0.0


@pytest.mark.parametrize("mu", [0.1, 1.0, 40.0, 800.0, 8000.0, 9e5])
def test_poisson_vs_mpmath(mu):
    lo, hi = oracle.band(mu, 10 ** 6)
    ks = sorted(set([lo, hi, (lo + hi) // 2, int(mu), max(lo, int(mu) - 3), min(hi, int(mu) + 7)]))
    for k in ks:
        ref = float(_mp_pois(k, mu))
        got = oracle.poisson_pmf(k, mu)
        assert abs(got - ref) <= 2e-15 * ref, (mu, k, got, ref)


def test_poisson_ratio_recurrence():
    # F(k+1)/F(k) = mu/(k+1): pins the exponent and the factorial index
    for mu in [3.7, 250.0, 123456.5]:
        lo, hi = oracle.band(mu, 10 ** 6)
        for k in range(lo, min(hi, lo + 50)):
            a, b = oracle.poisson_pmf(k, mu), oracle.poisson_pmf(k + 1, mu)
            assert b / a == pytest.approx(mu / (k + 1), rel=1e-13)


def _band_closed_form(mu, M, c=6.0, m=16):
    if mu == 0.0:
        return 0, 0
    s = math.sqrt(mu)
    lo = max(0, math.floor(mu - c * s))
    hi = min(M - 1, math.ceil(mu + c * s) + m)
    return lo, hi


@pytest.mark.parametrize("mu,M,expect", [
    (0.0, 50, (0, 0)), (0.1, 10 ** 6, (0, 18)), (1.0, 10 ** 6, (0, 23)),
    (40.0, 50, (2, 49)),            # hi = ceil(40 + 6*sqrt(40)) + 16 = 94 clipped to M-1
    (800.0, 10 ** 6, (630, 986)), (8000.0, 10 ** 6, (7463, 8553)),
    (9e5, 10 ** 6, (894307, 905709))])
def test_band_edges(mu, M, expect):
    # DESIGN.md reading R1: hand-derivable integers (e.g. 800 - 6*28.28 = 630.29 -> 630)
    assert oracle.band(mu, M) == expect == _band_closed_form(mu, M)


def test_band_edges_sweep_closed_form():
    rng = np.random.default_rng(5)
    for mu in np.concatenate([rng.uniform(0, 50, 200), np.geomspace(0.01, 9e5, 300)]):
        assert oracle.band(mu, 10 ** 6) == _band_closed_form(float(mu), 10 ** 6)


@pytest.mark.parametrize("mu,M", [(40.0, 50), (9e5, 10 ** 6), (1.0, 10 ** 6), (800.0, 10 ** 6)])
def test_row_mass(mu, M):
    # stored mass of a band row = P(lo <= X <= hi), X ~ Poisson(mu): regularized incomplete
    # gamma (mpmath), independent of the pmf summation.
    F = oracle.Probes(np.array([mu]), M)
    lo, hi = int(F.lo[0]), int(F.hi[0])
    mass = F.val.sum()
    cdf = lambda k: mpmath.gammainc(k + 1, mpmath.mpf(mu), mpmath.inf, regularized=True)
    ref = cdf(hi) - (cdf(lo - 1) if lo > 0 else 0)
    assert abs(mass - float(ref)) <= 1e-14 + 1e-14 * len(F.val) * 1e-2
    if (mu, M) == (40.0, 50):
        assert float(ref) == pytest.approx(0.92966493334060487, abs=1e-15)


def test_build_probes_tables():
    a2 = np.array([0.0, 0.5, 3.0, 10.0, 30.0])
    F = oracle.Probes(a2, 40)
    assert F.off[0] == 0 and np.all(np.diff(F.off) == F.len)
    for d, mu in enumerate(a2):
        lo, hi = oracle.band(mu, 40)
        assert (F.lo[d], F.hi[d]) == (lo, hi)
        for j in range(F.len[d]):
            assert F.val[F.off[d] + j] == oracle.poisson_pmf(lo + j, mu)
    assert np.all(F.val >= 0)


# ----------------------------------------------------------------------------- P8 projection
@pytest.mark.parametrize("x,y", [
    ([0.3, 0.7], [0.3, 0.7]), ([2.0, 0.0], [1.0, 0.0]),
    ([0.5, 0.4, 0.3], [0.5 - 0.2 / 3, 0.4 - 0.2 / 3, 0.3 - 0.2 / 3]),
    ([-1.0, -1.0], [0.5, 0.5]), ([5.0], [1.0]), ([0.0, 0.0, 0.0, 0.0], [0.25] * 4)])
def test_projection_examples(x, y):
    # PAPER.md:494-497 definition; examples are closed-form (symmetric / single threshold)
    got, _ = oracle.project_simplex(x)
    np.testing.assert_allclose(got, y, rtol=0, atol=1e-15)


def _brute_projection(x):
    """argmin_{y in S} ||x - y||: enumerate supports, keep the feasible KKT point."""
    n = len(x)
    best = None
    for r in range(1, n + 1):
        for S in itertools.combinations(range(n), r):
            tau = (sum(x[i] for i in S) - 1.0) / r
            y = np.zeros(n)
            for i in S:
                y[i] = x[i] - tau
            if y.min() < -1e-14:
                continue
            if any(x[i] > tau + 1e-14 for i in range(n) if i not in S):
                continue
            d = np.sum((x - y) ** 2)
            if best is None or d < best[0]:
                best = (d, y)
    return best[1]


def test_projection_brute_force_and_properties():
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 7))
        x = rng.normal(0, 1.0, n) * rng.choice([0.1, 1, 10])
        y, tau = oracle.project_simplex(x)
        np.testing.assert_allclose(y, _brute_projection(x), atol=1e-12)
        # KKT of the projection: y = max(x - tau, 0), sum y = 1, y >= 0
        assert y.min() >= 0 and abs(y.sum() - 1) <= 4 * n * 2.2e-16 * max(1.0, np.abs(x).max())
        np.testing.assert_allclose(y, np.maximum(x - tau, 0), atol=0)
        # idempotence, shift invariance
        np.testing.assert_allclose(oracle.project_simplex(y)[0], y, atol=1e-15)
        np.testing.assert_allclose(oracle.project_simplex(x + 3.25)[0], y, atol=1e-13)
        # non-expansiveness
        z = x + rng.normal(0, 0.5, n)
        assert np.linalg.norm(oracle.project_simplex(z)[0] - y) <= np.linalg.norm(z - x) + 1e-14


def test_project_rows():
    rng = np.random.default_rng(3)
    X = rng.normal(size=(100, 5))
    Y = oracle.project_rows(X)
    for k in range(100):
        np.testing.assert_array_equal(Y[k], oracle.project_simplex(X[k])[0])


# ----------------------------------------------------------------------------- P6, P7
def _micro(seed=0, D=12, M=9, N=4, mu_max=6.0):
    rng = np.random.default_rng(seed)
    a2 = np.sort(rng.uniform(0, mu_max, D))
    F = oracle.Probes(a2, M)
    Th = oracle.project_rows(rng.normal(0.3, 0.4, (M, N)))
    P = rng.dirichlet(np.ones(N), size=D)
    return F, Th, P


def _dense_L(M):
    Dm = np.diff(np.eye(M), axis=0)        # (M-1) x M forward difference
    return Dm.T @ Dm


def test_forward_backward_dense():
    # Table 1 rows objective / gradient against dense numpy
    for seed in range(4):
        F, Th, P = _micro(seed)
        Fd = F.dense()
        R = oracle.forward(F, Th, P)
        np.testing.assert_allclose(R, Fd @ Th - P, rtol=0, atol=1e-14)
        for gamma in [0.0, 0.37]:
            G = oracle.backward(F, R, Th, gamma)
            np.testing.assert_allclose(G, Fd.T @ R + gamma * _dense_L(F.M) @ Th, atol=1e-14)


def test_adjointness():
    rng = np.random.default_rng(7)
    F, Th, _ = _micro(1, D=30, M=40, N=3, mu_max=30)
    Rr = rng.normal(size=(F.D, 3))
    lhs = np.sum(oracle.forward(F, Th) * Rr)
    rhs = np.sum(Th * oracle.backward(F, Rr, Th, 0.0))
    assert lhs == pytest.approx(rhs, rel=1e-13)


def test_gradient_finite_difference():
    # grad f = 2G (reading R0): central differences of the objective (eq. min_obj2 + regul)
    rng = np.random.default_rng(11)
    F, Th, P = _micro(2)
    gamma = 0.05
    R = oracle.forward(F, Th, P)
    G = oracle.backward(F, R, Th, gamma)
    h = 1e-6
    for _ in range(20):
        k, n = int(rng.integers(F.M)), int(rng.integers(Th.shape[1]))
        E = np.zeros_like(Th)
        E[k, n] = h
        fd = (oracle.objective(F, P, Th + E, gamma) - oracle.objective(F, P, Th - E, gamma)) / (2 * h)
        assert fd == pytest.approx(2 * G[k, n], rel=1e-6, abs=1e-9)


def test_gradient_zero_at_exact_fit():
    F, Th, _ = _micro(3)
    P = F.dense() @ Th
    G = oracle.backward(F, oracle.forward(F, Th, P), Th, 0.0)
    assert np.abs(G).max() <= 1e-15


def test_stencil_and_regulariser():
    # constant columns -> L Theta = 0; f(Theta, g) - f(Theta, 0) = g * regul (eq. regul)
    M, N = 7, 3
    C = np.tile(np.array([0.2, 0.5, 0.3]), (M, 1))
    assert np.abs(oracle.laplacian(C)).max() == 0.0
    F, Th, P = _micro(4)
    g = 0.123
    reg = np.sum(np.diff(Th, axis=0) ** 2)
    assert oracle.regul(Th) == pytest.approx(reg, rel=1e-14)
    assert oracle.objective(F, P, Th, g) - oracle.objective(F, P, Th, 0.0) == pytest.approx(
        g * reg, rel=1e-12)
    # toy objective (SPEC-style): F = [1] (mu = 0 -> F_{0,0} = 1), P = [0.3], Theta = [0.7]
    F1 = oracle.Probes(np.array([0.0]), 1)
    assert oracle.objective(F1, np.array([[0.3]]), np.array([[0.7]]), 0.0) == pytest.approx(0.16)
    # M = 1: no regulariser
    assert oracle.regul(np.array([[0.4, 0.6]])) == 0.0


# ----------------------------------------------------------------------------- P4, P5
def test_sqs_majorizer():
    # w = F^T (F 1) + 4 gamma (reading R2) and diag(w) - (F^T F + gamma L) is PSD
    for seed, gamma in [(0, 0.0), (1, 1e-2), (2, 1.0)]:
        F, _, _ = _micro(seed, D=10, M=6, N=2)
        Fd = F.dense()
        w = oracle.sqs_weights(F, gamma)
        np.testing.assert_allclose(w, Fd.T @ (Fd @ np.ones(F.M)) + 4 * gamma, rtol=1e-14)
        ev = np.linalg.eigvalsh(np.diag(w) - (Fd.T @ Fd + gamma * _dense_L(F.M)))
        assert ev.min() >= -1e-12


def test_power_iteration_tiny():
    I = qs.tiny()
    F = oracle.Probes(I.alpha2, I.M)
    Fd = F.dense()
    lam = np.linalg.eigvalsh(Fd.T @ Fd).max()
    rho = oracle.power_iteration(F, 100)
    assert rho == pytest.approx(lam, rel=1e-6)
    assert rho <= oracle.sqs_weights(F, 0.0).max() * (1 + 1e-12)


# ----------------------------------------------------------------------------- KKT measure
def test_kkt_measure_closed_form():
    # PAPER.md:565-567 with df = 2G, N = 2, M = 3.
    # Row 0: Theta = (.25, .75), df = (1.4, 1.4): unclamped lambda = -1.4 -> 0;
    #        clamped lambda = 0 -> 1.96 * (.0625 + .5625) = 1.225.
    # Row 1: Theta = (1, 0), df = (-2, 4): lambda = 2 (both) -> 0.
    # Row 2: Theta = (.5, .5), df = (2, 6): unclamped lambda = -2 -> 0 + 4 = 4;
    #        clamped lambda = 0 -> 1 + 9 = 10.
    Th = np.array([[0.25, 0.75], [1.0, 0.0], [0.5, 0.5]])
    G = np.array([[0.7, 0.7], [-1.0, 2.0], [1.0, 3.0]])
    r, rp = oracle.kkt(Th, G)
    assert r == pytest.approx(math.sqrt(4 / 6), rel=1e-14)
    assert rp == pytest.approx(math.sqrt(11.225 / 6), rel=1e-14)


# ----------------------------------------------------------------------------- P9 .. P13
@pytest.mark.parametrize("step", [oracle.STEP_SQS, oracle.STEP_LIPSCHITZ])
def test_iteration_invariants(step):
    I = qs.tiny()
    F = oracle.Probes(I.alpha2, I.M)
    prev = None
    for k in [1, 2, 5, 20, 60]:
        r = oracle.solve(F, I.P, I.gamma, 0.0, k, step=step)
        Th = r["theta"]
        assert Th.min() >= 0.0
        assert np.abs(Th.sum(axis=1) - 1).max() <= 4 * Th.shape[1] * 2.2e-16
        tr = r["trace"]
        assert np.all(tr[1:] <= tr[:-1] * (1 + 1e-12))       # majorisation -> monotone descent
        if prev is not None:
            np.testing.assert_array_equal(tr[:len(prev)], prev)   # same path, prefix-stable
        prev = tr
    assert r["trace"][0] == pytest.approx(oracle.objective(F, I.P, np.full((I.M, 10), 0.1), I.gamma))


def test_fixed_point_noiseless():
    I = qs.tiny()
    F = oracle.Probes(I.alpha2, I.M)
    T = I.theta_true
    P = oracle.forward(F, T)
    r = oracle.solve(F, P, 0.0, 0.0, 100, theta0=T)
    assert np.abs(r["theta"] - T).max() <= 1e-13


def _brute_qp(Fd, P, gamma):
    """Exact QP optimum by active-set enumeration: for each support pattern solve the
    equality-constrained KKT system; keep the primal- and dual-feasible point."""
    D, M = Fd.shape
    N = P.shape[1]
    A = np.kron(Fd, np.eye(N))
    B = np.kron(np.diff(np.eye(M), axis=0), np.eye(N)) if M > 1 else np.zeros((0, M * N))
    H = 2 * (A.T @ A + gamma * B.T @ B)
    c = 2 * A.T @ P.ravel()
    C = np.kron(np.eye(M), np.ones((1, N)))
    sols = []
    for pat in itertools.product(range(1, 2 ** N), repeat=M):
        S = np.array([[(p >> n) & 1 for n in range(N)] for p in pat], bool).ravel()
        idx = np.nonzero(S)[0]
        m = len(idx)
        K = np.zeros((m + M, m + M))
        K[:m, :m] = H[np.ix_(idx, idx)]
        K[:m, m:] = C[:, idx].T
        K[m:, :m] = C[:, idx]
        try:
            z = np.linalg.solve(K, np.concatenate([c[idx], np.ones(M)]))
        except np.linalg.LinAlgError:
            continue
        th = np.zeros(M * N)
        th[idx] = z[:m]
        if th.min() < -1e-13:
            continue
        g = H @ th - c
        lam = z[m:]
        if all(S[k * N + n] or g[k * N + n] >= -lam[k] - 1e-11 for k in range(M)
               for n in range(N)):
            sols.append((th.reshape(M, N), g.reshape(M, N)))
    return sols


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("gamma", [0.0, 1e-3, 1e-2])
def test_exact_qp_optimum(seed, gamma):
    rng = np.random.default_rng(100 + seed)
    M, N, D = 4, 3, 8
    F = oracle.Probes(np.sort(rng.uniform(0.3, 3.0, D)), M)
    P = rng.dirichlet(np.ones(N), size=D)
    sols = _brute_qp(F.dense(), P, gamma)
    assert len(sols) == 1
    th_star, g_star = sols[0]
    for accel, iters in [(0, 50000), (1, 20000)]:
        r = oracle.solve(F, P, gamma, 0.0, iters, accel=accel)
        np.testing.assert_allclose(r["theta"], th_star, atol=1e-12)
    # P12: KKT at convergence -- on-support df equals the row minimum, off-support df >= it
    G = oracle.backward(F, oracle.forward(F, r["theta"], P), r["theta"], gamma)
    for k in range(M):
        mn = G[k].min()
        for n in range(N):
            if th_star[k, n] > 1e-9:
                assert G[k, n] == pytest.approx(mn, abs=1e-10 * max(1, abs(mn)))
            else:
                assert G[k, n] >= mn - 1e-12
    np.testing.assert_allclose(2 * G, g_star, atol=1e-10)
    assert oracle.kkt(r["theta"], G)[0] <= 1e-12


def _fidelity(pi, pt):
    # eq. fidelities for diagonal operators: (sum sqrt(p q))^2 / (sum p sum q)
    return np.sum(np.sqrt(pi * pt)) ** 2 / (pi.sum() * pt.sum())


def test_noiseless_recovery_tiny():
    # P13: data-space recovery on noiseless Tiny; fidelity bar of PAPER.md:133 (> 99%)
    I = qs.tiny()
    F = oracle.Probes(I.alpha2, I.M)
    P = oracle.forward(F, I.theta_true)
    r = oracle.solve(F, P, 0.0, 0.0, 1000, accel=1, kkt_every=50)
    normP = np.sum(P ** 2)
    assert r["trace"][-1] <= 1e-10 * normP
    fid = [_fidelity(r["theta"][:, n], I.theta_true[:, n]) for n in range(P.shape[1])]
    assert min(fid) >= 0.98 and np.mean(fid) >= 0.99


def test_early_stop_semantics():
    # reading R3: stop at the first k with r(Theta_k) <= tol and return Theta_k
    I = qs.tiny()
    F = oracle.Probes(I.alpha2, I.M)
    full = oracle.solve(F, I.P, I.gamma, 0.0, 40)
    tol = full["kkt"][25] * 1.0000001
    k = int(np.nonzero(full["kkt"] <= tol)[0][0])
    r = oracle.solve(F, I.P, I.gamma, tol, 40)
    assert r["iters_done"] == k
    ref = oracle.solve(F, I.P, I.gamma, 0.0, k)
    np.testing.assert_array_equal(r["theta"], ref["theta"])


# ----------------------------------------------------------------------------- P14 synth
def test_tiny_ground_truth_rows():
    T = qs.theta_tiny()
    np.testing.assert_allclose(T[0], np.eye(10)[0], atol=1e-15)
    np.testing.assert_allclose(T[1, :2], [0.2, 0.8], atol=1e-15)
    np.testing.assert_allclose(T[2, :3], [0.04, 0.32 + 0.64 / 9, 0.64 * 8 / 9], atol=1e-15)
    np.testing.assert_allclose(T.sum(axis=1), 1.0, atol=1e-13)
    assert T.min() >= 0


def test_medium_ground_truth_rows():
    T = qs.theta_medium(50, 10)
    np.testing.assert_allclose(T[1, :2], [0.1, 0.9], atol=1e-15)
    np.testing.assert_allclose(T.sum(axis=1), 1.0, atol=1e-12)


def test_objective_sum_accuracy_many_terms():
    # f = ||F Theta - P||^2 over 2e6 entries vs an exactly rounded sum (math.fsum) of the
    # dense residual: the accumulation must stay within the reading-R5 gate (1e-10) by far.
    rng = np.random.default_rng(21)
    D, M, N = 2000, 200, 1000
    F = oracle.Probes(np.sort(rng.uniform(0, 150, D)), M)
    Th = np.full((M, N), 1.0 / N)
    P = rng.dirichlet(np.ones(N) * 0.05, D)
    R = F.dense() @ Th - P
    ref = math.fsum((R * R).ravel())
    assert oracle.objective(F, P, Th, 0.0) == pytest.approx(ref, rel=1e-14)


# ----------------------------------------------------------------------------- smoothing (f4)
def test_smoothing_pins():
    """eq. smoothing, reading R13: closed forms and invariants."""
    rng = np.random.default_rng(8)
    M, N = 400, 5
    Th = oracle.project_rows(rng.normal(0.2, 0.3, (M, N)))
    S = oracle.smooth(Th, exclude=100, div=50)
    # rows below the exclusion are untouched; every row stays on the simplex (convex combination)
    np.testing.assert_array_equal(S[:100], Th[:100])
    assert S.min() >= 0 and np.abs(S.sum(1) - 1).max() <= 1e-13
    # brute force of the definition with numpy (window [i - i//50, i + i//50] clipped to [0, M))
    for i in [100, 149, 150, 250, 399]:
        ns = i // 50
        lo, hi = max(0, i - ns), min(M - 1, i + ns)
        np.testing.assert_allclose(S[i], Th[lo:hi + 1].mean(0), rtol=1e-14, atol=1e-16)
    # i = 150: Ns = 3, window rows 147..153 (7 rows, the paper's 2 Ns + 1)
    np.testing.assert_allclose(S[150], Th[147:154].sum(0) / 7, rtol=1e-14)
    # a column that is linear in i is reproduced where the window is symmetric (no clipping)
    L = np.tile(np.arange(M, dtype=float)[:, None], (1, 2))
    SL = oracle.smooth(L, exclude=0, div=50)
    interior = [i for i in range(M) if i + i // 50 <= M - 1]
    np.testing.assert_allclose(SL[interior], L[interior], rtol=1e-14)
    # constant columns are fixed points; div <= 0 disables the smoothing
    C = np.full((M, 3), 1.0 / 3)
    np.testing.assert_allclose(oracle.smooth(C), C, rtol=1e-15)
    np.testing.assert_array_equal(oracle.smooth(Th, div=0), Th)


# ----------------------------------------------------------------------------- BB step (R14)
@pytest.mark.parametrize("gamma", [1e-3, 1e-2])
def test_bb_reaches_exact_qp_optimum(gamma):
    """Barzilai-Borwein scalar step (reading R14) converges to the brute-force QP optimum (P11)."""
    rng = np.random.default_rng(300)
    M, N, D = 4, 3, 8
    F = oracle.Probes(np.sort(rng.uniform(0.3, 3.0, D)), M)
    P = rng.dirichlet(np.ones(N), size=D)
    sols = _brute_qp(F.dense(), P, gamma)
    assert len(sols) == 1
    r = oracle.solve(F, P, gamma, 0.0, 3000, step=oracle.STEP_BB)
    np.testing.assert_allclose(r["theta"], sols[0][0], atol=1e-12)
    # the first step is the Lipschitz step, so iteration 1 matches LIPSCHITZ exactly
    r1 = oracle.solve(F, P, gamma, 0.0, 1, step=oracle.STEP_BB)
    l1 = oracle.solve(F, P, gamma, 0.0, 1, step=oracle.STEP_LIPSCHITZ)
    np.testing.assert_array_equal(r1["theta"], l1["theta"])


def test_bb_step_formula():
    """Iteration 2 of BB uses t = <s,s>/(||F s||^2 + gamma ||D s||^2), s = Theta_1 - Theta_0:
    reproduce it with dense numpy from the oracle's own iterates."""
    rng = np.random.default_rng(301)
    F = oracle.Probes(np.sort(rng.uniform(0.2, 6.0, 10)), 7)
    P = rng.dirichlet(np.ones(4), 10)
    g = 0.05
    th0 = np.full((7, 4), 0.25)
    th1 = oracle.solve(F, P, g, 0.0, 1, step=oracle.STEP_BB)["theta"]
    s = th1 - th0
    Fd = F.dense()
    Ds = np.diff(s, axis=0)
    t = np.sum(s * s) / (np.sum((Fd @ s) ** 2) + g * np.sum(Ds * Ds))
    rho = oracle.power_iteration(F, 100)
    tl = 1.0 / (1.01 * rho + 4 * g)
    t = min(max(t, tl), 1e6 * tl)
    G1 = oracle.backward(F, oracle.forward(F, th1, P), th1, g)
    th2 = oracle.project_rows(th1 - t * G1)
    np.testing.assert_allclose(oracle.solve(F, P, g, 0.0, 2, step=oracle.STEP_BB)["theta"], th2,
                               atol=1e-14)


# ---------------------------------------------------------------------------- FISTA (P13 gap)
def _np_project_rows(X):
    """Sort-based Euclidean projection of every row onto the simplex, written here in NumPy."""
    U = -np.sort(-X, axis=1)
    css = np.cumsum(U, axis=1) - 1.0
    j = np.arange(1, X.shape[1] + 1)
    rho = (U - css / j > 0).sum(axis=1)
    tau = css[np.arange(X.shape[0]), rho - 1] / rho
    return np.maximum(X - tau[:, None], 0.0)


def _np_L(T):
    """(L Theta) of eq. regul with free ends (reading R8), dense NumPy."""
    L = np.zeros_like(T)
    L[1:] += T[1:] - T[:-1]
    L[:-1] += T[:-1] - T[1:]
    return L


def test_fista_coefficients_beck_teboulle():
    """Iterations 1-3 of the oracle's SQS-FISTA equal a dense NumPy run of the Beck-Teboulle
    recurrence tau_{k+1} = (1 + sqrt(1 + 4 tau_k^2)) / 2, beta_k = (tau_k - 1) / tau_{k+1},
    Y_k = Theta_k + beta_k (Theta_k - Theta_{k-1}) (SURVEY 8(c) algorithm step 4.1), with the
    SQS step of reading R2; a plausible wrong recurrence beta_k = (tau_k - 1) / tau_k misses."""
    rng = np.random.default_rng(11)
    M, N, D, gamma = 30, 4, 25, 1e-3
    a2 = np.sort(rng.uniform(0.0, 22.0, D))
    F = oracle.Probes(a2, M)
    A = F.dense()
    P = rng.dirichlet(np.ones(N), D)
    w = A.T @ (A @ np.ones(M)) + 4.0 * gamma
    t = 1.0 / w

    def run(beta_of, K):
        th = np.full((M, N), 1.0 / N)
        prev = th.copy()
        tau = 1.0
        out = []
        for _ in range(K):
            tn = (1.0 + np.sqrt(1.0 + 4.0 * tau * tau)) / 2.0
            b = beta_of(tau, tn)
            Y = th + b * (th - prev)
            G = A.T @ (A @ Y - P) + gamma * _np_L(Y)
            prev, th = th, _np_project_rows(Y - t[:, None] * G)
            tau = tn
            out.append(th)
        return out

    good = run(lambda tau, tn: (tau - 1.0) / tn, 3)
    wrong = run(lambda tau, tn: (tau - 1.0) / tau, 3)
    for k in (1, 2, 3):
        ref = oracle.solve(F, P, gamma, 0.0, k, accel=1)
        np.testing.assert_allclose(ref["theta"], good[k - 1], rtol=0, atol=1e-13)
        if k >= 2:   # beta_0 = 0 either way; from k = 2 the sequences separate
            assert np.abs(ref["theta"] - wrong[k - 1]).max() > 1e-6
    # the returned resume state: tau_3 and Theta_2
    r3 = oracle.solve(F, P, gamma, 0.0, 3, accel=1)
    tau = 1.0
    for _ in range(3):
        tau = (1.0 + np.sqrt(1.0 + 4.0 * tau * tau)) / 2.0
    assert r3["fista_t"] == tau
    np.testing.assert_allclose(r3["theta_prev"], good[1], rtol=0, atol=1e-13)


def test_fista_resume_continues_the_sequence():
    """solve(K1) then solve(K2) from (Theta_K1, Theta_K1-1, tau_K1) is the uninterrupted
    solve(K1 + K2) bit for bit (the resume state of SURVEY 8(b))."""
    rng = np.random.default_rng(12)
    M, N, D, gamma = 40, 5, 30, 1e-3
    F = oracle.Probes(np.sort(rng.uniform(0.0, 30.0, D)), M)
    P = rng.dirichlet(np.ones(N), D)
    full = oracle.solve(F, P, gamma, 0.0, 9, accel=1)
    a = oracle.solve(F, P, gamma, 0.0, 4, accel=1)
    b = oracle.solve(F, P, gamma, 0.0, 5, accel=1, theta0=a["theta"], theta_prev=a["theta_prev"],
                     fista_t=a["fista_t"])
    assert np.array_equal(b["theta"], full["theta"])
    assert np.array_equal(b["trace"], full["trace"][4:])
    # a fresh restart from Theta_4 (momentum reset) is a different sequence
    c = oracle.solve(F, P, gamma, 0.0, 5, accel=1, theta0=a["theta"])
    assert np.abs(c["theta"] - full["theta"]).max() > 1e-9


# ------------------------------------------------------------- BB + exact line search (R17)
@pytest.mark.parametrize("gamma", [1e-3, 1e-2])
def test_bb_line_search_qp_optimum_and_monotone(gamma):
    """BB with the exact line search along the projected direction (reading
    R17) converges to the brute-force QP optimum (P11) and, unlike the unsafeguarded BB step,
    never increases f (an exact minimisation along a feasible direction)."""
    rng = np.random.default_rng(310)
    M, N, D = 4, 3, 8
    F = oracle.Probes(np.sort(rng.uniform(0.3, 3.0, D)), M)
    P = rng.dirichlet(np.ones(N), size=D)
    sols = _brute_qp(F.dense(), P, gamma)
    r = oracle.solve(F, P, gamma, 0.0, 3000, step=oracle.STEP_BB_LS)
    np.testing.assert_allclose(r["theta"], sols[0][0], atol=1e-12)
    tr = r["trace"]
    assert np.all(tr[1:] <= tr[:-1] * (1 + 1e-13) + 1e-300)


def test_bb_line_search_step_formula():
    """Iteration 2 of BB-LS reproduced in dense NumPy: BB t from s = Theta_1 - Theta_0, Z =
    P_S(Theta_1 - t G), d = Z - Theta_1, l* = clip(-<G,d> / (||F d||^2 + gamma ||D d||^2), 0, 1)
    from the quadratic f(Theta + l d) (no oracle function on the path except the pinned
    forward / backward / projection)."""
    rng = np.random.default_rng(311)
    F = oracle.Probes(np.sort(rng.uniform(0.2, 6.0, 10)), 7)
    P = rng.dirichlet(np.ones(4), 10)
    g = 0.05
    A = F.dense()

    def f(T):
        return float(np.sum((A @ T - P) ** 2) + g * np.sum(np.diff(T, axis=0) ** 2))

    th0 = np.full((7, 4), 0.25)
    rho = oracle.power_iteration(F, 100)
    tl = 1.0 / (1.01 * rho + 4 * g)
    th = [th0]
    for k in range(2):   # two iterations by hand
        T = th[-1]
        G = A.T @ (A @ T - P) + g * _np_L(T)
        if k == 0:
            t = tl
        else:
            s = th[-1] - th[-2]
            t = np.sum(s * s) / (np.sum((A @ s) ** 2) + g * np.sum(np.diff(s, axis=0) ** 2))
            t = min(max(t, tl), 1e6 * tl)
        d = _np_project_rows(T - t * G) - T
        den = np.sum((A @ d) ** 2) + g * np.sum(np.diff(d, axis=0) ** 2)
        assert -np.sum(G * d) >= np.sum(d * d) / t * (1 - 1e-12)   # projection property
        lam = min(max(max(-np.sum(G * d), np.sum(d * d) / t) / den, 0.0), 1.0)
        nxt = T + lam * d
        # l* is the exact minimiser of f along d on [0, 1]
        for l2 in (0.0, 1.0, lam * 0.9, min(1.0, lam * 1.1)):
            assert f(nxt) <= f(T + l2 * d) + 1e-15
        th.append(nxt)
    r = oracle.solve(F, P, g, 0.0, 2, step=oracle.STEP_BB_LS)
    np.testing.assert_allclose(r["theta"], th[2], atol=1e-13)
