"""Input generators (qdt_synth) pinned on CPU: the paper-shaped detector workload (SURVEY 8(f)
row 2) must produce the analytic POVM of PAPER.md:200-219, and the fidelity report must follow
eq. fidelities in its diagonal form."""
import itertools

import numpy as np
import pytest

import qdt_synth as qs


def test_click_probs_closed_forms():
    """eq. pj_fock at i = 0 (no clicks), i = 1 (the per-photon probabilities of eq. pj_coh's
    exponents: R eta_det for j = 1, (1-R)^2/R (R eta_loop)^(j-1) eta_det after)."""
    R, el, ed = qs.TMD_R, qs.TMD_ETA_LOOP, qs.TMD_ETA_DET
    p = qs.tmd_click_probs(np.array([0, 1, 7]), bins=5)
    assert np.all(p[0] == 0)
    ref1 = [R * ed] + [(1 - R) ** 2 / R * (R * el) ** (j - 1) * ed for j in range(2, 6)]
    np.testing.assert_allclose(p[1], ref1, rtol=1e-14)
    np.testing.assert_allclose(p[2], 1 - (1 - np.array(ref1)) ** 7, rtol=1e-13)


def test_povm_against_brute_force_enumeration():
    """Poisson binomial by enumerating all 2^bins click patterns (bins = 6)."""
    bins = 6
    rows = np.array([0, 1, 3, 40, 500])
    p = qs.tmd_click_probs(rows, bins)
    T = qs.theta_tmd(501, bins=bins)[rows]
    for r in range(len(rows)):
        ref = np.zeros(bins + 1)
        for pat in itertools.product((0, 1), repeat=bins):
            ref[sum(pat)] += np.prod([p[r, j] if c else 1 - p[r, j] for j, c in enumerate(pat)])
        np.testing.assert_allclose(T[r], ref, rtol=1e-12, atol=1e-300)


def test_povm_moments_and_shape():
    """Rows are distributions over N = 151 outcomes with the Poisson-binomial mean sum_j p_j and
    variance sum_j p_j (1 - p_j); Theta_0 = e_0 (vacuum never clicks)."""
    T = qs.theta_tmd(3000, block=700)
    assert T.shape == (3000, 151) and T.min() >= 0
    np.testing.assert_allclose(T.sum(1), 1.0, atol=1e-13)
    assert T[0, 0] == 1.0
    n = np.arange(151)
    p = qs.tmd_click_probs(np.arange(3000))
    mean = T @ n
    np.testing.assert_allclose(mean, p.sum(1), rtol=1e-11, atol=1e-13)
    var = T @ (n * n) - mean ** 2
    np.testing.assert_allclose(var, (p * (1 - p)).sum(1), rtol=1e-8, atol=1e-11)


def test_paper_tmd_shape():
    """Quadratic probes |alpha_d|^2 = d^2; D = 1076 reaches the paper's M ~ 1.2e6."""
    I = qs.paper_tmd(40, noiseless=True)
    assert I.N == 151 and I.D == 40
    np.testing.assert_array_equal(I.alpha2, np.arange(40.0) ** 2)
    assert I.M > 39 ** 2 + 5 * 39
    np.testing.assert_allclose(I.P.sum(1), 1.0, atol=1e-9)   # nothing leaks past the cutoff
    D = 1076
    mu = (D - 1) ** 2
    assert 1.15e6 < int(mu + 6 * np.sqrt(mu) + 100) < 1.25e6


def test_fidelity_definition():
    a = np.array([[0.5, 0.0], [0.5, 1.0]])
    assert np.allclose(qs.fidelities(a, a), 1.0)
    b = np.array([[1.0, 0.0], [0.0, 1.0]])
    # column 0: (sqrt(.5))^2 / (1 * 1) = 0.5; column 1: (sqrt(1))^2 / (1 * 1) = 1
    np.testing.assert_allclose(qs.fidelities(a, b), [0.5, 1.0])
    assert qs.fidelities(3 * a, a) == pytest.approx([1.0, 1.0])   # scale invariant


def test_logbins_rowwise_builder_matches_binwise():
    """theta_logbins_rows (vectorised, used at Stress size) builds exactly the Theta_true of the
    bin-by-bin theta_logbins_sparse."""
    for M, N in [(3000, 300), (5000, 1200)]:
        A = qs.theta_logbins_sparse(M, N)
        B = qs.theta_logbins_rows(M, N, chunk=777)
        assert A.shape == B.shape and A.nnz == B.nnz
        assert abs(A - B).max() == 0.0
        assert np.allclose(np.asarray(B.sum(1)).ravel(), 1.0, atol=1e-14)
