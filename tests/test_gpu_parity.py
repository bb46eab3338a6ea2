"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element
on the same seeded inputs (-m gpu).  Tolerances:
  band edges, counts, indices            exact
  F values                               4 eps (8 + |ln F|) relative (exp conditioning)
  R, G, projections (single op)          1e-13 x scale (fp64 sums in a different order)
  Theta after identical iteration counts 1e-9 max-abs      (north_star)
  objective trace                        1e-10 relative + cancellation floor (reading R5)
"""
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
    return q


@pytest.fixture(scope="module")
def ctx(q):
    return q.qdt_init(0)


def _trace_ok(tg, to, P):
    tg, to = np.asarray(tg), np.asarray(to)
    floor = 4 * EPS * np.sqrt(np.sum(P ** 2)) * np.sqrt(np.abs(to))
    return np.all(np.abs(tg - to) <= 1e-10 * np.abs(to) + floor + 1e-300)


# ----------------------------------------------------------------------------- S0 probes
@pytest.mark.parametrize("name", ["tiny", "medium", "edge"])
def test_probe_parity(q, ctx, name):
    if name == "edge":
        a2 = np.array([0.0, 0.0, 1e-3, 0.1, 1.0, 15.9, 16.0, 16.1, 39.9, 40.0, 77.0, 120.0, 500.0])
        M = 100
    else:
        I = getattr(qs, name)()
        a2, M = I.alpha2, I.M
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    ex = q.qdt_probes_export(ctx, Fg)
    np.testing.assert_array_equal(ex["lo"], Fo.lo)
    np.testing.assert_array_equal(ex["len"], Fo.len)
    assert ex["nnz"] == Fo.nnz
    # F = exp(l): a relative error of F is an absolute error of l = ln F, so the bound scales
    # with |ln F| (a few ulps of the log's magnitude)
    tol = 4 * EPS * (8 + np.abs(np.log(np.maximum(Fo.val, 1e-300))))
    bad = np.nonzero(np.abs(ex["val"] - Fo.val) > tol * Fo.val)[0]
    if bad.size:
        i = bad[np.argmax(np.abs(ex["val"] - Fo.val)[bad] / Fo.val[bad])]
        d = int(np.searchsorted(Fo.off, i, side="right") - 1)
        k = int(Fo.lo[d] + i - Fo.off[d])
        pytest.fail(f"{bad.size} values off; worst mu={a2[d]!r} k={k} gpu={ex['val'][i]!r} "
                    f"oracle={Fo.val[i]!r} rel={abs(ex['val'][i] / Fo.val[i] - 1):.3e}")


def test_probe_parity_megascale_edges_and_sample(q, ctx):
    a2 = np.geomspace(1.0, 9e5, 10 ** 4)
    M = 10 ** 6
    Fg = q.qdt_build_probes(ctx, a2, M)
    ex = q.qdt_probes_export(ctx, Fg)
    lo_hi = np.array([oracle.band(m, M) for m in a2])
    np.testing.assert_array_equal(ex["lo"], lo_hi[:, 0])
    np.testing.assert_array_equal(ex["len"], lo_hi[:, 1] - lo_hi[:, 0] + 1)
    off = np.concatenate([[0], np.cumsum(ex["len"])])
    rng = np.random.default_rng(0)
    for d in rng.choice(10 ** 4, 60, replace=False):
        for j in rng.choice(ex["len"][d], 5):
            ref = oracle.poisson_pmf(ex["lo"][d] + j, a2[d])
            assert abs(ex["val"][off[d] + j] - ref) <= 4 * EPS * (8 + abs(np.log(ref))) * ref


# ----------------------------------------------------------------------------- S5 projection
@pytest.mark.parametrize("N", [1, 2, 10, 31, 32, 33, 100, 257, 1000])
def test_projection_parity(q, ctx, N):
    rng = np.random.default_rng(N)
    X = rng.normal(0, 1, (300, N)) * rng.choice([0.01, 1, 30], (300, 1))
    X[0] = 0.0
    X[1] = 1.0 / N
    Yg = q.qdt_project_rows(ctx, X)
    Yo = oracle.project_rows(X)
    scale = np.maximum(1.0, np.abs(X).max(axis=1, keepdims=True))
    assert np.all(np.abs(Yg - Yo) <= 1e-14 * N * scale)
    assert Yg.min() >= 0


# ----------------------------------------------------------------------------- S2, S3, S4
def _cases():
    out = []
    for name in ["tiny", "medium"]:
        I = getattr(qs, name)()
        out.append((name, I.alpha2, I.M, I.P, I.gamma))
    for seed, (D, M, N) in enumerate([(1, 1, 1), (3, 7, 5), (50, 333, 17), (400, 97, 100),
                                      (3000, 64, 10), (20, 2000, 3)]):
        I = qs.random_instance(seed, D, M, N)
        out.append((f"rand{D}x{M}x{N}", I.alpha2, I.M, I.P, I.gamma))
    # many low-mu probes: every tile window is wider than the split cap (split-K path)
    rng = np.random.default_rng(9)
    a2 = np.sort(rng.uniform(0, 6, 2500))
    out.append(("splitK", a2, 40, rng.dirichlet(np.ones(100), 2500), 1e-3))
    return out


CASES = _cases()


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_residual_gradient_parity(q, ctx, case):
    _, a2, M, P, gamma = case
    N = P.shape[1]
    rng = np.random.default_rng(1)
    Th = oracle.project_rows(rng.normal(0.5, 0.5, (M, N)))
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    Ro = oracle.forward(Fo, Th, P)
    Rg = q.qdt_residual(ctx, Fg, Th, P)
    sR = max(1.0, np.abs(P).max())
    assert np.abs(Rg - Ro).max() <= 1e-13 * sR
    Go = oracle.backward(Fo, Ro, Th, gamma)
    Gg = q.qdt_gradient(ctx, Fg, Ro, Th, gamma)
    sG = max(1.0, np.abs(Go).max())
    assert np.abs(Gg - Go).max() <= 1e-13 * sG


@pytest.mark.parametrize("case", CASES[:4], ids=[c[0] for c in CASES[:4]])
def test_step_setup_parity(q, ctx, case):
    _, a2, M, P, gamma = case
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    w, rho = q.qdt_step_setup(ctx, Fg, gamma, 100)
    np.testing.assert_allclose(w, oracle.sqs_weights(Fo, gamma), rtol=1e-13)
    assert rho == pytest.approx(oracle.power_iteration(Fo, 100), rel=1e-12)


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("step", [0, 1])
def test_one_step_parity(q, ctx, case, step):
    _, a2, M, P, gamma = case
    N = P.shape[1]
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    Th = np.full((M, N), 1.0 / N)
    ro = oracle.solve(Fo, P, gamma, 0.0, 1, step=step)
    rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 1, step=step, use_graph=False)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-12
    assert _trace_ok(rg["trace"], ro["trace"], P)
    del Th


# ----------------------------------------------------------------------------- full solves
@pytest.mark.parametrize("step,accel,iters", [(0, 0, 2000), (1, 0, 2000), (0, 1, 2000)])
def test_tiny_solve_parity(q, ctx, step, accel, iters):
    I = qs.tiny()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    ke = 50 if accel else 1
    ro = oracle.solve(Fo, I.P, I.gamma, 0.0, iters, step=step, accel=accel, kkt_every=ke)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, iters, step=step, accel=bool(accel),
                     kkt_every=ke)
    assert rg["info"]["iters_done"] == ro["iters_done"] == iters
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], I.P)
    m = ~np.isnan(ro["kkt"])
    np.testing.assert_array_equal(m, ~np.isnan(rg["kkt"]))
    np.testing.assert_allclose(rg["kkt"][m], ro["kkt"][m], rtol=1e-8, atol=1e-15)
    # P9 invariants on the GPU iterate
    Th = rg["theta"]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 4 * Th.shape[1] * EPS
    if not accel:
        tr = rg["trace"]
        assert np.all(tr[1:] <= tr[:-1] * (1 + 1e-12))


@pytest.mark.parametrize("accel", [0, 1])
def test_medium_solve_parity(q, ctx, accel):
    I = qs.medium()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    iters = 200
    ro = oracle.solve(Fo, I.P, I.gamma, 0.0, iters, accel=accel, kkt_every=10 if accel else 1)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, iters, accel=bool(accel),
                     kkt_every=10 if accel else 1)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], I.P)


def test_early_stop_parity(q, ctx):
    I = qs.tiny()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    full = oracle.solve(Fo, I.P, I.gamma, 0.0, 300)
    tol = full["kkt"][137] * (1 + 1e-7)
    ro = oracle.solve(Fo, I.P, I.gamma, tol, 300)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, tol, 300, check_every=16)
    assert rg["info"]["iters_done"] == ro["iters_done"]
    assert rg["info"]["converged"] == 1
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-12


def test_splitk_and_uncovered_rows(q, ctx):
    # low-mu probes only: rows above the bands are uncovered (reading R9); gamma = 0 freezes
    # them at 1/N, gamma > 0 diffuses them.  Windows exceed the split cap (split-K fix-up).
    rng = np.random.default_rng(4)
    a2 = np.sort(rng.uniform(0, 8, 1500))
    M, N = 120, 33
    P = rng.dirichlet(np.ones(N), 1500)
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    for gamma in [0.0, 1e-2]:
        ro = oracle.solve(Fo, P, gamma, 0.0, 150)
        rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 150)
        assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
        assert rg["info"]["uncovered_rows"] == M - 1 - Fo.hi.max()
        if gamma == 0.0:
            assert np.all(rg["theta"][Fo.hi.max() + 1:] == 1.0 / N)


def test_deterministic_and_device_pointers(q, ctx):
    torch = pytest.importorskip("torch")
    I = qs.medium()
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    a = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 50)
    b = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 50)
    np.testing.assert_array_equal(a["theta"], b["theta"])
    np.testing.assert_array_equal(a["trace"], b["trace"])
    Pd = torch.tensor(I.P, device="cuda")
    c = q.qdt_solve(ctx, Fg, Pd, I.gamma, 0.0, 50)
    np.testing.assert_array_equal(c["theta"].cpu().numpy(), a["theta"])
    f, r = q.qdt_objective(ctx, Fg, I.P, a["theta"], I.gamma)
    Fo = oracle.Probes(I.alpha2, I.M)
    assert f == pytest.approx(oracle.objective(Fo, I.P, a["theta"], I.gamma), rel=1e-12)


def test_error_paths(q, ctx):
    with pytest.raises(q.QdtError, match="UNSORTED"):
        q.qdt_build_probes(ctx, np.array([1.0, 0.5]), 10)
    with pytest.raises(q.QdtError, match="INVALID_ARG"):
        q.qdt_build_probes(ctx, np.array([-1.0]), 10)
    with pytest.raises(q.QdtError, match="INVALID_ARG"):
        q.qdt_build_probes(ctx, np.array([1.0]), 0)
    with pytest.raises(q.QdtError, match="TRUNCATED"):
        q.qdt_build_probes(ctx, np.array([40.0]), 50, strict_mass=True)
    F = q.qdt_build_probes(ctx, np.array([1.0, 2.0]), 10)
    P = np.full((2, 3), 1 / 3)
    P[1, 1] = np.nan
    with pytest.raises(q.QdtError, match="NONFINITE"):
        q.qdt_solve(ctx, F, P, 0.0, 0.0, 5)
    with pytest.raises(q.QdtError, match="INVALID_ARG"):
        q.qdt_solve(ctx, F, np.full((2, 3), 1 / 3), -1.0, 0.0, 5)


@pytest.mark.slow
def test_large_solve_parity(q, ctx):
    I = qs.large()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    ro = oracle.solve(Fo, I.P, I.gamma, 0.0, 3)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 3)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], I.P)


@pytest.mark.slow
def test_megascale_solve_parity(q, ctx):
    """Full-size bench workload, same launch configuration as bench.py (graph replay)."""
    I = qs.megascale()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    ro = oracle.solve(Fo, I.P, I.gamma, 0.0, 2)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 2, use_graph=True)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], I.P)
    Th = rg["theta"]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 4 * Th.shape[1] * EPS


@pytest.mark.parametrize("N,gamma", [(20, 1e-3), (37, 0.0), (100, 1e-5), (8, 1e-2)])
def test_long_axis_sweep_parity(q, ctx, N, gamma):
    """Log-spaced probes over a long Fock axis: most tiles have narrow windows beside a few split
    heavy tiles; 30 iterations against the oracle, P9 invariants, trace."""
    rng = np.random.default_rng(N)
    D, M = 400, 30000
    a2 = np.geomspace(1.0, 0.9 * M, D)
    P = rng.dirichlet(np.ones(N) * 0.3, D)
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    ro = oracle.solve(Fo, P, gamma, 0.0, 30)
    rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 30)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], P)
    np.testing.assert_allclose(rg["kkt"], ro["kkt"], rtol=1e-8, atol=1e-15)
    Th = rg["theta"]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 4 * N * EPS


@pytest.mark.parametrize("N,kkt_every", [(100, 1), (37, 5), (8, 3)])
def test_fista_sweep_parity(q, ctx, N, kkt_every):
    """SQS-FISTA on the sweep kernels (Theta_{k-1} tile staged beside Theta_k, Y formed in the
    epilogue, device-gated KKT evaluation pass) against the oracle's FISTA, 40 iterations."""
    rng = np.random.default_rng(100 + N)
    D, M = 300, 20000
    a2 = np.geomspace(1.0, 0.9 * M, D)
    P = rng.dirichlet(np.ones(N) * 0.3, D)
    gamma = 1e-4
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    ro = oracle.solve(Fo, P, gamma, 0.0, 40, accel=1, kkt_every=kkt_every)
    rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 40, accel=True, kkt_every=kkt_every)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], P)
    m = ~np.isnan(ro["kkt"])
    np.testing.assert_array_equal(m, ~np.isnan(rg["kkt"]))
    np.testing.assert_allclose(rg["kkt"][m], ro["kkt"][m], rtol=1e-8, atol=1e-15)


@pytest.mark.slow
def test_stress_cut_solve_parity(q, ctx):
    """Stress-shaped cut-down instance (M = 10^5, N = 10^3, D = 2000 log-spaced
    probes, log bins, noiseless P): N > 128 runs the general kernels; 3 iterations."""
    I = qs.stress_cut()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    ro = oracle.solve(Fo, I.P, I.gamma, 0.0, 3)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 3)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], I.P)
    Th = rg["theta"]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 4 * Th.shape[1] * EPS


@pytest.mark.parametrize("N,accel", [(200, 0), (1000, 0), (151, 0), (250, 1), (151, 1), (129, 0),
                                     (1023, 0), (152, 0), (160, 0), (137, 0), (162, 0)])
def test_wide_sweep_parity(q, ctx, N, accel):
    """N > 128: the wide sweep (balanced column-chunk DMMA gradient + warp-per-row projection +
    column-chunked forward), plain and FISTA; plain steps at N <= 160 take k_bwd_mma with 17-20
    n-blocks instead; odd N (151, the paper's outcome count) runs on a row pitch N + 1 with a
    zero pad column excluded from the projection and the KKT.  25 iterations against the
    oracle."""
    rng = np.random.default_rng(N)
    D, M = 300, 6000
    a2 = np.geomspace(0.5, 0.9 * M, D)
    P = rng.dirichlet(np.ones(N) * 0.2, D)
    gamma = 1e-3
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    ro = oracle.solve(Fo, P, gamma, 0.0, 25, accel=accel, kkt_every=5 if accel else 1)
    rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 25, accel=bool(accel), kkt_every=5 if accel else 1)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], P)
    m = ~np.isnan(ro["kkt"])
    np.testing.assert_allclose(rg["kkt"][m], ro["kkt"][m], rtol=1e-8, atol=1e-15)
    f, r = q.qdt_objective(ctx, Fg, P, rg["theta"], gamma)
    assert f == pytest.approx(oracle.objective(Fo, P, rg["theta"], gamma), rel=1e-12)


@pytest.mark.parametrize("D,M,N", [(1, 1, 1), (1, 5, 128), (7, 40, 129), (9, 50, 130), (5, 300, 16),
                                   (40, 64, 8), (40, 65, 8), (12, 130, 1)])
def test_shape_edges(q, ctx, D, M, N):
    """Boundary shapes: single probe / Fock row / outcome, the sweep's N limit (128 | 129 odd ->
    general kernels | 130 even -> wide sweep), tile-multiple and tile-plus-one M, N = 1; probe means
    beyond the cutoff (bands clipped to the last row) and repeated means."""
    rng = np.random.default_rng(D * 1000 + M * 10 + N)
    a2 = np.sort(np.concatenate([rng.uniform(0, 1.5 * M, D - D // 3), np.full(D // 3, 0.5 * M)]))
    P = rng.dirichlet(np.ones(N), D) if N > 1 else np.ones((D, 1))
    gamma = 1e-2
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    for accel in (0, 1):
        ro = oracle.solve(Fo, P, gamma, 0.0, 12, accel=accel)
        rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 12, accel=bool(accel))
        assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9, accel
        assert _trace_ok(rg["trace"], ro["trace"], P)
        Th = rg["theta"]
        assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 4 * max(N, 2) * EPS


@pytest.mark.parametrize("M,N,exclude,div", [(400, 5, 100, 50), (3000, 100, 100, 50), (257, 8, 0, 7),
                                             (1000, 33, 1001, 50), (50, 4, 10, 0)])
def test_smoothing_parity(q, ctx, M, N, exclude, div):
    """Long-range smoothing (reading R13) against the oracle; host and device."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(M + N)
    Th = oracle.project_rows(rng.normal(0.2, 0.4, (M, N)))
    ref = oracle.smooth(Th, exclude, div)
    got = q.qdt_smooth(ctx, Th, exclude, div)
    assert np.abs(got - ref).max() <= 1e-13
    gd = q.qdt_smooth(ctx, torch.tensor(Th, device="cuda"), exclude, div)
    np.testing.assert_array_equal(gd.cpu().numpy(), got)


def test_smooth_then_restart_parity(q, ctx):
    """The paper's refinement: solve, smooth, second solve from the smoothed
    matrix (warm start through theta0), against the same sequence on the oracle."""
    I = qs.medium()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    r1o = oracle.solve(Fo, I.P, I.gamma, 0.0, 60, accel=1, kkt_every=10)
    r1g = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 60, accel=True, kkt_every=10)
    so, sg = oracle.smooth(r1o["theta"]), q.qdt_smooth(ctx, r1g["theta"])
    assert np.abs(sg - so).max() <= 1e-9
    r2o = oracle.solve(Fo, I.P, I.gamma, 0.0, 40, theta0=so)
    r2g = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 40, theta0=sg)
    assert np.abs(r2g["theta"] - r2o["theta"]).max() <= 1e-9
    assert _trace_ok(r2g["trace"], r2o["trace"], I.P)


def test_bb_step_parity(q, ctx):
    """Barzilai-Borwein step (reading R14): the first iterates match the oracle's BB iterates; at
    convergence both reach the unique QP minimiser (gamma > 0, brute-force optimum of P11)."""
    import itertools  # noqa: F401
    from test_oracle_pins import _brute_qp
    rng = np.random.default_rng(300)
    M, N, D = 4, 3, 8
    a2 = np.sort(rng.uniform(0.3, 3.0, D))
    P = rng.dirichlet(np.ones(N), size=D)
    gamma = 1e-2
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    star = _brute_qp(Fo.dense(), P, gamma)[0][0]
    rg = q.qdt_solve(ctx, Fg, P, gamma, 0.0, 3000, step=q.QDT_STEP_BB)
    assert np.abs(rg["theta"] - star).max() <= 1e-9
    I = qs.tiny()
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    ro = oracle.solve(Fo, I.P, I.gamma, 0.0, 8, step=oracle.STEP_BB)
    rg = q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 8, step=q.QDT_STEP_BB)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    assert _trace_ok(rg["trace"], ro["trace"], I.P)
    assert rg["info"]["step_scalar"] == pytest.approx(ro["step"], rel=1e-12)
    # long runs diverge iterate-wise (roundoff amplification, reading R5) but reach the same
    # minimiser on a well-conditioned instance (gamma > 0)
    rng = np.random.default_rng(302)
    a2 = np.sort(rng.uniform(0.0, 12.0, 60))
    P = rng.dirichlet(np.ones(6), 60)
    Fo = oracle.Probes(a2, 20)
    Fg2 = q.qdt_build_probes(ctx, a2, 20)
    ro = oracle.solve(Fo, P, 1e-2, 0.0, 4000, step=oracle.STEP_BB)
    rg = q.qdt_solve(ctx, Fg2, P, 1e-2, 0.0, 4000, step=q.QDT_STEP_BB)
    assert ro["kkt"][-1] <= 1e-12 and rg["kkt"][-1] <= 1e-12
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    with pytest.raises(q.QdtError, match="INVALID_ARG"):
        q.qdt_solve(ctx, Fg, I.P, I.gamma, 0.0, 5, step=q.QDT_STEP_BB, accel=True)


def test_odd_wide_theta0_device_and_objective(q, ctx):
    """Padded-pitch odd N through every entry: host theta0, device P/theta0/out, qdt_objective."""
    import torch
    rng = np.random.default_rng(7)
    D, M, N = 90, 1500, 151
    a2 = np.geomspace(0.5, 0.9 * M, D)
    P = rng.dirichlet(np.ones(N) * 0.3, D)
    th0 = rng.dirichlet(np.ones(N), M)
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    ro = oracle.solve(Fo, P, 1e-3, 0.0, 12, theta0=th0)
    rg = q.qdt_solve(ctx, Fg, P, 1e-3, 0.0, 12, theta0=th0)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    Pd = torch.tensor(P, device="cuda")
    td = torch.tensor(th0, device="cuda")
    rd = q.qdt_solve(ctx, Fg, Pd, 1e-3, 0.0, 12, theta0=td)
    th = rd["theta"].cpu().numpy() if hasattr(rd["theta"], "cpu") else rd["theta"]
    assert np.array_equal(th, rg["theta"])
    f, r = q.qdt_objective(ctx, Fg, P, ro["theta"], 1e-3)
    assert f == pytest.approx(oracle.objective(Fo, P, ro["theta"], 1e-3), rel=1e-12)
    # early stop on the KKT tolerance: same stopping iteration (post-stop evaluation pass)
    full = oracle.solve(Fo, P, 1e-3, 0.0, 80)
    tol = full["kkt"][41] * (1 + 1e-7)
    ro2 = oracle.solve(Fo, P, 1e-3, tol, 80)
    rg2 = q.qdt_solve(ctx, Fg, P, 1e-3, tol, 80, check_every=16)
    assert rg2["info"]["iters_done"] == ro2["iters_done"] and rg2["info"]["converged"] == 1
    assert np.abs(rg2["theta"] - ro2["theta"]).max() <= 1e-9
    R = oracle.forward(Fo, ro["theta"], P)
    G = oracle.backward(Fo, R, ro["theta"], 1e-3)
    assert r == pytest.approx(oracle.kkt(ro["theta"], G)[0], rel=1e-8)


def test_paper_tmd_parity(q, ctx):
    """The paper's detector workload shape: quadratic probes, N = 151
    outcomes of the analytic time-multiplexed-detector POVM, multinomial noise; D = 60."""
    I = qs.paper_tmd(60)
    Fo = oracle.Probes(I.alpha2, I.M)
    Fg = q.qdt_build_probes(ctx, I.alpha2, I.M)
    for accel in (0, 1):
        ro = oracle.solve(Fo, I.P, 1e-4, 0.0, 20, accel=accel, kkt_every=5 if accel else 1)
        rg = q.qdt_solve(ctx, Fg, I.P, 1e-4, 0.0, 20, accel=bool(accel), kkt_every=5 if accel else 1)
        assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
        assert _trace_ok(rg["trace"], ro["trace"], I.P)


# ------------------------------------------------------------------ 8(f) row 1: Newton solve
@pytest.mark.parametrize("seed,D,M,N,gamma,conv", [(1, 30, 60, 5, 1e-3, 1), (2, 20, 30, 3, 1e-2, 1),
                                                   (3, 80, 40, 6, 1e-4, 1), (4, 200, 700, 37, 1e-4, 0),
                                                   (5, 120, 80, 151, 1e-3, 0), (6, 120, 80, 200, 1e-3, 0)])
def test_newton_parity(q, ctx, seed, D, M, N, gamma, conv):
    """qdt_solve_newton against the oracle's or_newton (reading R16): the first iterations
    step for step (same stage, CG count and step length; Theta to 1e-9), then (well-posed
    cases) the same minimiser (objective 1e-12 relative) at the KKT tolerance; the
    ill-conditioned case (M > D, small gamma) only step for step."""
    rng = np.random.default_rng(seed)
    a2 = np.sort(rng.uniform(0.0, 0.8 * M, D))
    P = rng.dirichlet(np.ones(N), D)
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    for k in (1, 3):
        ro = oracle.newton(Fo, P, gamma, k)
        rg = q.qdt_solve_newton(ctx, Fg, P, gamma, 0.0, k)
        assert rg["info"]["iters_done"] == ro["iters_done"]
        np.testing.assert_array_equal(rg["stage"], ro["stage"])
        np.testing.assert_array_equal(rg["cg"], ro["cg"])
        np.testing.assert_allclose(rg["alpha"], ro["alpha"], rtol=0)
        assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
        assert _trace_ok(rg["trace"], ro["trace"], P)
    if not conv:
        return
    ro = oracle.newton(Fo, P, gamma, 400, eps_kkt=1e-12)
    rg = q.qdt_solve_newton(ctx, Fg, P, gamma, 1e-12, 400)
    assert rg["kkt"][-1] <= 1e-12
    assert rg["trace"][-1] == pytest.approx(ro["trace"][-1], rel=1e-12)
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-6
    Th = rg["theta"]
    assert Th.min() >= 0 and np.abs(Th.sum(1) - 1).max() <= 1e-12


def test_newton_theta0_and_errors(q, ctx):
    """Newton from a given start (a few PG iterations) matches the oracle from the same start;
    bad options are rejected."""
    rng = np.random.default_rng(9)
    D, M, N, gamma = 40, 50, 4, 1e-3
    a2 = np.sort(rng.uniform(0.0, 40.0, D))
    P = rng.dirichlet(np.ones(N), D)
    Fo = oracle.Probes(a2, M)
    Fg = q.qdt_build_probes(ctx, a2, M)
    th0 = oracle.solve(Fo, P, gamma, 0.0, 20)["theta"]
    ro = oracle.newton(Fo, P, gamma, 4, theta0=th0)
    rg = q.qdt_solve_newton(ctx, Fg, P, gamma, 0.0, 4, theta0=th0)
    np.testing.assert_array_equal(rg["cg"], ro["cg"])
    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
    with pytest.raises(q.QdtError):
        q.qdt_solve_newton(ctx, Fg, P, gamma, 0.0, 4, cg_max=0)


def test_graph_cache_keys(q, ctx):
    """The solve loop's CUDA graph is reused across calls with the same key (configuration,
    handle ids, device buffers); alternating handles / gammas / lengths must each match the
    oracle, and a repeated call must reproduce its first result bitwise."""
    rng = np.random.default_rng(11)
    D, M, N = 120, 400, 12
    cases = []
    for j in range(2):
        a2 = np.sort(rng.uniform(0.0, 0.8 * M, D))
        cases.append((a2, rng.dirichlet(np.ones(N), D)))
    Fg = [q.qdt_build_probes(ctx, a2, M) for a2, _ in cases]
    first = {}
    for rep in range(2):
        for j, (a2, P) in enumerate(cases):
            for gamma, iters in ((1e-3, 40), (1e-4, 33)):
                rg = q.qdt_solve(ctx, Fg[j], P, gamma, 0.0, iters, use_graph=True)
                key = (j, gamma, iters)
                if rep == 0:
                    ro = oracle.solve(oracle.Probes(a2, M), P, gamma, 0.0, iters)
                    assert np.abs(rg["theta"] - ro["theta"]).max() <= 1e-9
                    first[key] = rg["theta"].copy()
                else:
                    assert np.array_equal(rg["theta"], first[key])
