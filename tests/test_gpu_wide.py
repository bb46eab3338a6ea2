"""GPU parity of the fused wide step (csrc/qdt_wide.cu, N > 128: thread-block clusters of up
to 16 CTAs per 32-row Fock tile, cluster-wide Michelot through distributed shared memory)
against the oracle (-m gpu).  Shapes cross the cluster-size choices (1 .. 16 CTAs), odd N on
the padded pitch, ragged tiles, the Stress row width N = 10^4, and (slow) the Stress-shaped
M = 10^5 x N = 10^4 instance of SURVEY 8(c)."""
import numpy as np
import pytest

import oracle
import qdt_synth as qs

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16


@pytest.fixture(scope="module")
def q():
    import paper_2404_02844_b200 as q
    from paper_2404_02844_b200 import build
    build.build()
    oracle.set_threads(0)
    return q


@pytest.fixture(scope="module")
def ctx(q):
    return q.qdt_init(0)


@pytest.fixture(autouse=True)
def fused_wide(monkeypatch):
    """Every plan built in these tests takes the fused wide step, also at 128 < N <= 1024 (where the
    two-kernel sweep is the default)."""
    monkeypatch.setenv("QDT_WIDE", "new")


def _trace_ok(tg, to, P):
    tg, to = np.asarray(tg), np.asarray(to)
    floor = 4 * EPS * np.sqrt(np.sum(P ** 2)) * np.sqrt(np.abs(to))
    return np.all(np.abs(tg - to) <= 1e-10 * np.abs(to) + floor + 1e-300)


def _check(q, ctx, a2, M, P, gamma, iters, accel=0, kkt_every=1, theta0=None):
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    ro = oracle.solve(Fo, P, gamma, 0.0, iters, accel=accel, kkt_every=kkt_every, theta0=theta0)
    rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, iters, accel=bool(accel), kkt_every=kkt_every, theta0=theta0)
    d = np.abs(rg["theta"] - ro["theta"]).max()
    assert d <= 1e-9, d
    assert _trace_ok(rg["trace"], ro["trace"], P)
    m = np.isfinite(ro["kkt"])
    np.testing.assert_allclose(rg["kkt"][m], ro["kkt"][m], rtol=1e-8, atol=1e-15)
    Th = rg["theta"]
    N = P.shape[1]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 8 * N * EPS
    return rg


@pytest.mark.parametrize("N,accel", [(1500, 0), (2048, 0), (4096, 0), (10000, 0), (2048, 1), (1501, 0),
                                     (700, 1), (641, 0), (10240, 0)])
def test_wide_shapes(q, ctx, N, accel):
    """N in {1 500, 2 048, 4 096, 10^4}, odd N, the 640-column CTA boundary, the widest
    row of the build; M = 900 leaves a ragged last tile; log-spaced probes."""
    rng = np.random.default_rng(N)
    D, M = 120, 900
    a2 = np.geomspace(0.3, 0.85 * M, D)
    P = rng.dirichlet(np.ones(N) * 0.2, D)
    _check(q, ctx, a2, M, P, 1e-4, 6, accel=accel, kkt_every=2 if accel else 1)


def test_wide_early_stop_and_objective(q, ctx):
    rng = np.random.default_rng(3)
    D, M, N = 100, 700, 2000
    a2 = np.sort(rng.uniform(0, 0.8 * M, D))
    P = rng.dirichlet(np.ones(N) * 0.3, D)
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    full = oracle.solve(Fo, P, 1e-3, 0.0, 60)
    tol = full["kkt"][33] * (1 + 1e-7)
    ro = oracle.solve(Fo, P, 1e-3, tol, 60)
    rg = q.qdt_solve(ctx, Fg, P, 1e-3, tol, 60, check_every=16)
    assert rg["info"]["iters_done"] == ro["iters_done"] and rg["info"]["converged"] == 1
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    f, r = q.qdt_objective(ctx, Fg, P, ro["theta"], 1e-3)
    assert f == pytest.approx(oracle.objective(Fo, P, ro["theta"], 1e-3), rel=1e-12)
    G = oracle.backward(Fo, oracle.forward(Fo, ro["theta"], P), ro["theta"], 1e-3)
    assert r == pytest.approx(oracle.kkt(ro["theta"], G)[0], rel=1e-8)


def test_wide_deterministic(q, ctx):
    rng = np.random.default_rng(5)
    D, M, N = 150, 2000, 3000
    a2 = np.geomspace(1.0, 0.8 * M, D)
    P = rng.dirichlet(np.ones(N) * 0.2, D)
    Fg = q.qdt_build_probes(ctx, a2, M)
    a = q.qdt_solve(ctx, Fg, P, 1e-4, 0.0, 20)
    b = q.qdt_solve(ctx, Fg, P, 1e-4, 0.0, 20)
    assert np.array_equal(a["theta"], b["theta"]) and np.array_equal(a["trace"], b["trace"])


@pytest.mark.slow
@pytest.mark.parametrize("accel", [0, 1])
def test_stress_shaped_parity(q, ctx, accel):
    """SURVEY 8(c) Stress row: the Stress generator at M = 10^5, N = 10^4, D = 2000 (noiseless
    P = F Theta_true, log bins, gamma = 1e-5), 3 iterations, plain and FISTA."""
    I = qs.stress(M=10 ** 5, N=10 ** 4, D=2000)
    _check(q, ctx, I.alpha2, I.M, I.P, I.gamma, 3, accel=accel)
