"""oracle-MT: the oracle's OpenMP split leaves every floating-point operation
and its order unchanged and sums every reduction in a fixed chunk order, so results are
bit-identical for any thread count.  Checked on shapes that span several row blocks / chunks."""
import numpy as np
import pytest

import oracle
import qdt_synth as qs


@pytest.fixture
def restore_threads():
    yield
    oracle.set_threads(0)


def _run_all(F, P, gamma, accel, step):
    r = oracle.solve(F, P, gamma, 0.0, 6, step=step, accel=accel)
    G = oracle.backward(F, oracle.forward(F, r["theta"], P), r["theta"], gamma)
    return r, G, oracle.sqs_weights(F, gamma), oracle.objective(F, P, r["theta"], gamma)


@pytest.mark.parametrize("accel,step", [(0, oracle.STEP_SQS), (1, oracle.STEP_SQS), (0, oracle.STEP_BB)])
def test_bitwise_identical_across_thread_counts(restore_threads, accel, step):
    rng = np.random.default_rng(3)
    M, N, D = 1300, 7, 400                      # > 5 backward row blocks, > 1 reduction chunk
    F = oracle.Probes(np.sort(rng.uniform(0.0, 1100.0, D)), M)
    P = rng.dirichlet(np.ones(N), D)
    oracle.set_threads(1)
    assert oracle.get_threads() == 1
    r1, G1, w1, f1 = _run_all(F, P, 1e-4, accel, step)
    oracle.set_threads(4)
    assert oracle.get_threads() == 4
    r4, G4, w4, f4 = _run_all(F, P, 1e-4, accel, step)
    assert np.array_equal(r1["theta"], r4["theta"])
    assert np.array_equal(r1["trace"], r4["trace"])
    assert np.array_equal(r1["kkt"], r4["kkt"], equal_nan=True)
    assert np.array_equal(G1, G4) and np.array_equal(w1, w4) and f1 == f4


def test_newton_identical_across_thread_counts(restore_threads):
    I = qs.tiny()
    F = oracle.Probes(I.alpha2, I.M)
    oracle.set_threads(1)
    a = oracle.newton(F, I.P, I.gamma, 6)
    oracle.set_threads(3)
    b = oracle.newton(F, I.P, I.gamma, 6)
    assert np.array_equal(a["theta"], b["theta"]) and np.array_equal(a["alpha"], b["alpha"])
