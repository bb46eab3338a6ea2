"""Pins of the oracle's two-stage two-metric projected truncated Newton (
PAPER.md:458-567; reading R16).  Each piece is checked against dense linear algebra written
here from the definitions (not against itself): the Hessian diagonal of Table 1, the masked
Newton systems of eq. 2metric D / I (stage 1) and of the transformed variables of Alg. 1
(stage 2), the one-sided arc derivatives by finite differences, and the full solve against
the projected-gradient oracle's minimiser on well-posed instances."""
import numpy as np
import pytest

import oracle


def _instance(seed, D, M, N, gamma):
    rng = np.random.default_rng(seed)
    a2 = np.sort(rng.uniform(0.0, 0.8 * M, D))
    F = oracle.Probes(a2, M)
    P = rng.dirichlet(np.ones(N), D)
    return F, P, gamma


def _dense_H(F, gamma):
    """Per-column Hessian 2 (F^T F + gamma L), L = D^T D (forward differences, free ends)."""
    A = F.dense()
    M = F.M
    Dm = np.zeros((M - 1, M))
    for i in range(M - 1):
        Dm[i, i], Dm[i, i + 1] = -1.0, 1.0
    return 2.0 * (A.T @ A + gamma * Dm.T @ Dm)


def _grad(F, P, Theta, gamma):
    R = oracle.forward(F, Theta, P)
    return 2.0 * oracle.backward(F, R, Theta, gamma)


def test_hessian_diagonal_table1():
    F, P, g = _instance(0, 25, 40, 3, 1e-2)
    np.testing.assert_allclose(oracle.hess_diag(F, g), np.diag(_dense_H(F, g)), rtol=1e-13)


def test_stage1_direction_no_active_set_is_the_newton_step():
    """eps < 0 (no active set), CG to convergence: p solves H p = -df column by column."""
    F, P, g = _instance(1, 60, 30, 4, 1e-2)    # D > M: H nonsingular
    rng = np.random.default_rng(5)
    Th = rng.dirichlet(np.ones(4), 30)
    p, slope, it = oracle.newton_direction(F, P, g, Th, eps_active=-1.0, cg_max=400)
    H = _dense_H(F, g)
    df = _grad(F, P, Th, g)
    ref = np.linalg.solve(H, -df)
    # truncated CG stops at ||r|| <= min(.5, sqrt||b||)||b||: compare the residual, not p
    r = H @ p + df
    assert np.linalg.norm(r) <= min(0.5, np.sqrt(np.linalg.norm(df))) * np.linalg.norm(df) * (1 + 1e-9)
    assert it >= 1
    # CG to a tight relative residual: p is the exact Newton step
    p2, _, _ = oracle.newton_direction(F, P, g, Th, eps_active=-1.0, cg_max=400, cg_rtol=1e-13)
    np.testing.assert_allclose(p2, ref, rtol=1e-8, atol=1e-10 * np.abs(ref).max())
    assert np.all(np.isfinite(ref))


def test_stage1_direction_active_set():
    """Entries with Theta <= eps and df > 0 get p = -df / h_i; the others solve the Hessian
    restricted to the free set (eq. 2metric D)."""
    F, P, g = _instance(2, 50, 24, 3, 1e-2)
    rng = np.random.default_rng(6)
    Th = rng.dirichlet(np.ones(3), 24)
    Th[::3, 0] = 0.0
    Th /= Th.sum(1, keepdims=True)
    P = P * 0.0 + oracle.forward(F, Th) + 1e-10 * rng.standard_normal(P.shape)
    P[:, 0] -= 0.1   # make df > 0 on column 0 so the zeros are active
    df = _grad(F, P, Th, g)
    act = (Th <= 1e-8) & (df > 0)
    assert act.sum() >= 3
    p, _, _ = oracle.newton_direction(F, P, g, Th, eps_active=1e-8, cg_max=500, cg_rtol=1e-13)
    h = oracle.hess_diag(F, g)
    np.testing.assert_allclose(p[act], (-df / h[:, None])[act], rtol=1e-12)
    H = _dense_H(F, g)
    for n in range(3):
        fr = ~act[:, n]
        Hf = H[np.ix_(fr, fr)]
        ref = np.linalg.solve(Hf, -df[fr, n])
        np.testing.assert_allclose(p[fr, n], ref, rtol=1e-8, atol=1e-10 * np.abs(ref).max())


def test_stage2_direction_reduced_system():
    """Alg. 1 transformation: x = Theta without the row maxima; reduced gradient
    df_in - df_{i,m(i)}, reduced Hessian Z^T H Z (solved densely here)."""
    F, P, g = _instance(3, 40, 16, 3, 1e-2)
    rng = np.random.default_rng(7)
    Th = rng.dirichlet(np.ones(3), 16)
    P = oracle.forward(F, Th) + 1e-9 * rng.standard_normal(P.shape)
    m = oracle.row_argmax(Th)
    p, slope, _ = oracle.newton_direction(F, P, g, Th, m=m, eps_active=-1.0, cg_max=2000, cg_rtol=1e-13)
    M, N = Th.shape
    free = [(i, n) for i in range(M) for n in range(N) if n != m[i]]
    idx = {v: j for j, v in enumerate(free)}
    Z = np.zeros((M * N, len(free)))
    for (i, n), j in idx.items():
        Z[i * N + n, j] = 1.0
        Z[i * N + m[i], j] = -1.0
    H = np.kron(_dense_H(F, g), np.eye(N))       # (M N) x (M N), row-major Theta
    df = _grad(F, P, Th, g).ravel()
    ref = np.linalg.solve(Z.T @ H @ Z, -(Z.T @ df))
    got = np.array([p[i, n] for (i, n) in free])
    np.testing.assert_allclose(got, ref, rtol=1e-8, atol=1e-10 * np.abs(ref).max())
    assert np.all(p[np.arange(M), m] == 0.0)
    np.testing.assert_allclose(slope, (Z.T @ df) @ ref, rtol=1e-6)


def test_arc_derivatives_by_finite_differences():
    """stage 1: df . d0 is the one-sided derivative of f(P_S[Theta + a p]) at a = 0 (d0 the
    tangent-cone projection); stage 2: of f along the clamped arc of the reduced variables."""
    F, P, g = _instance(4, 40, 20, 4, 1e-3)
    rng = np.random.default_rng(8)
    Th = rng.dirichlet(np.ones(4) * 0.5, 20)
    Th[Th < 0.05] = 0.0
    Th /= Th.sum(1, keepdims=True)
    f0 = oracle.objective(F, P, Th, g)
    p, slope, _ = oracle.newton_direction(F, P, g, Th, eps_active=1e-8, cg_max=30)
    a = 1e-7
    fd = (oracle.objective(F, P, oracle.project_rows(Th + a * p), g) - f0) / a
    assert slope == pytest.approx(fd, rel=1e-4, abs=1e-9)
    m = oracle.row_argmax(Th)
    p2, slope2, _ = oracle.newton_direction(F, P, g, Th, m=m, eps_active=1e-8, cg_max=30)
    T1 = np.maximum(Th + a * p2, 0.0)
    T1[np.arange(20), m] = 0.0
    T1[np.arange(20), m] = 1.0 - T1.sum(1)
    fd2 = (oracle.objective(F, P, T1, g) - f0) / a
    assert slope2 == pytest.approx(fd2, rel=1e-4, abs=1e-9)


@pytest.mark.parametrize("seed,D,M,N,gamma", [(1, 30, 60, 5, 1e-3), (2, 20, 30, 3, 1e-2),
                                              (3, 80, 40, 6, 1e-4)])
def test_newton_reaches_the_projected_gradient_minimiser(seed, D, M, N, gamma):
    """Well-posed instances (strictly convex: D >= M or gamma > 0 with covered rows): the
    two-stage Newton and the PG oracle reach the same unique minimiser; Armijo makes the
    trace monotone; every accepted step keeps Theta on the simplex."""
    F, P, g = _instance(seed, D, M, N, gamma)
    r = oracle.newton(F, P, g, 400, eps_kkt=1e-12)
    ro = oracle.solve(F, P, g, 1e-15, 60000, accel=1, kkt_every=1)
    assert r["kkt"][-1] <= 1e-12
    # same objective to 1e-12; the iterates agree to the conditioning of the minimiser
    assert r["trace"][-1] == pytest.approx(ro["trace"][-1], rel=1e-12)
    assert np.abs(r["theta"] - ro["theta"]).max() <= 1e-6
    assert np.all(np.diff(r["trace"]) <= 1e-15 * r["trace"][0])
    Th = r["theta"]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 1e-13
    assert set(np.unique(r["stage"])) <= {1, 2}


def test_row_argmax_first_on_ties():
    T = np.array([[0.2, 0.4, 0.4], [1.0, 0.0, 0.0], [0.3, 0.3, 0.4]])
    np.testing.assert_array_equal(oracle.row_argmax(T), [1, 0, 2])


def _np_project_rows(X):
    U = -np.sort(-X, axis=1)
    css = np.cumsum(U, axis=1) - 1.0
    j = np.arange(1, X.shape[1] + 1)
    rho = (U - css / j > 0).sum(axis=1)
    tau = css[np.arange(X.shape[0]), rho - 1] / rho
    return np.maximum(X - tau[:, None], 0.0)


def _np_f(A, P, T, gamma):
    R = A @ T - P
    return float(np.sum(R * R) + gamma * np.sum((T[:-1] - T[1:]) ** 2))


@pytest.mark.parametrize("seed,D,M,N", [(10, 20, 40, 4), (12, 20, 40, 4), (10, 30, 24, 3)])
def test_line_search_is_the_papers_armijo_rule(seed, D, M, N):
    """armijo = 0: every accepted step length alpha_k = beta^m is the smallest m >= 0 with
    f(P[Theta + beta^m p]) <= f(Theta) + c beta^m slope (beta = 3/4,
    c = 1/10), slope the one-sided arc derivative at 0 (pinned by finite differences above);
    the objective and the arcs are re-evaluated here in dense NumPy.  Stage 2 arcs are the
    clamped transformed arcs of Alg. 1 (infeasible lengths are skipped)."""
    F, P, g = _instance(seed, D, M, N, 1e-3)
    A = F.dense()
    K = 8
    run = oracle.newton(F, P, g, K, armijo=0)
    ks = len(run["alpha"])
    assert ks >= 4
    seen = set()
    for k in range(ks):
        Th = oracle.newton(F, P, g, k, armijo=0)["theta"]
        Tn = oracle.newton(F, P, g, k + 1, armijo=0)["theta"]
        st, al = int(run["stage"][k]), float(run["alpha"][k])
        seen.add(st)
        m_acc = int(round(np.log(al) / np.log(0.75)))
        assert al == 0.75 ** m_acc
        if st == 1:
            p, slope, _ = oracle.newton_direction(F, P, g, Th)
            arc = lambda a: _np_project_rows(Th + a * p)
            T0 = Th
        else:
            m = oracle.row_argmax(Th)
            T0 = Th.copy()
            rows = np.arange(T0.shape[0])
            T0[rows, m] = 0.0
            T0[rows, m] = 1.0 - T0.sum(1)
            p, slope, _ = oracle.newton_direction(F, P, g, T0, m=m)

            def arc(a, T0=T0, p=p, m=m, rows=rows):
                T = np.maximum(T0 + a * p, 0.0)
                T[rows, m] = 0.0
                T[rows, m] = 1.0 - T.sum(1)
                return T if T[rows, m].min() >= 0.0 else None
        f0 = _np_f(A, P, T0, g)
        assert slope < 0.0
        T1 = arc(al)
        np.testing.assert_allclose(Tn, T1, rtol=0, atol=1e-13)
        assert _np_f(A, P, T1, g) <= f0 + 0.1 * al * slope + 1e-13 * abs(f0)
        for mm in range(m_acc):   # every shorter exponent (longer step) fails the test
            a = 0.75 ** mm
            Ta = arc(a)
            if Ta is None:
                continue
            assert _np_f(A, P, Ta, g) > f0 + 0.1 * a * slope - 1e-13 * abs(f0)
    # the secant form of R16 (armijo = 1) is a different rule: on the first two instances it
    # accepts other lengths (so the checks above discriminate the two)
    sec = oracle.newton(F, P, g, K, armijo=1)
    if M == 40:
        assert not np.array_equal(sec["alpha"][:ks], run["alpha"][:ks])
