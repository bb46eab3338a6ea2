"""Oracle pins against the worked values under tests/golden/ (-m "not gpu").  Every fixture
file cites the PAPER.md passage its values follow and shows the hand derivation."""
import os

import numpy as np
import pytest

import oracle

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _rows(name):
    for line in open(os.path.join(G, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            yield line


def test_golden_band_edges():
    n = 0
    for line in _rows("band_edges.txt"):
        mu, M, lo, hi = line.split()
        assert oracle.band(float(mu), int(M)) == (int(lo), int(hi)), line
        n += 1
    assert n == 7


def test_golden_projection_examples():
    for line in _rows("projection_examples.txt"):
        x, y = line.split("|")
        x = np.array([float(v) for v in x.split()])
        y = np.array([float(v) for v in y.split()])
        got, _ = oracle.project_simplex(x)
        np.testing.assert_allclose(got, y, rtol=0, atol=2e-16)


def test_golden_poisson_values():
    for line in _rows("poisson_values.txt"):
        kind, mu, k, v = line.split()
        if kind == "pmf":
            assert oracle.poisson_pmf(int(k), float(mu)) == pytest.approx(float(v), rel=1e-15,
                                                                          abs=0)
        else:
            F = oracle.Probes(np.array([float(mu)]), int(k))
            assert F.val.sum() == pytest.approx(float(v), abs=2e-15)


def test_golden_kkt_example():
    d = {}
    for line in _rows("kkt_example.txt"):
        key, *vals = line.split()
        d[key] = np.array([float(v) for v in vals])
    r, rp = oracle.kkt(d["theta"].reshape(3, 2), d["G"].reshape(3, 2))
    assert r == pytest.approx(d["r"][0], rel=1e-14)
    assert rp == pytest.approx(d["r_paper"][0], rel=1e-14)
