"""Pins for the TEPS arithmetic and root sampling."""
import numpy as np
import pytest

import oracle
from tests import graphs


def test_compute_teps_spec():
    assert oracle.compute_teps(1000, 0.001) == pytest.approx(1e6)
    assert oracle.compute_teps(0, 1.0) == 0
    with pytest.raises(ValueError):
        oracle.compute_teps(5, 0.0)


def test_harmonic_mean_spec():
    assert oracle.harmonic_mean([2, 6]) == pytest.approx(3)
    assert oracle.harmonic_mean([7.5, 7.5, 7.5]) == pytest.approx(7.5)
    assert oracle.harmonic_mean([1, 4, 4]) == pytest.approx(2)
    for bad in ([], [1, 0], [2, -1]):
        with pytest.raises(ValueError):
            oracle.harmonic_mean(bad)


def test_component_tuples():
    n, uv = graphs.g1()
    g = oracle.build_csr(n, uv)
    d, _ = oracle.bfs(g, 0)
    assert oracle.component_tuples(uv, d) == 5
    uv1 = np.array([[0, 1]], np.int32)
    g1 = oracle.build_csr(2, uv1)
    d1, _ = oracle.bfs(g1, 0)
    assert oracle.component_tuples(uv1, d1) == 1                       # 1 edge, not 2 arcs
    # duplicates and self-loops inside the component are counted (R5)
    uv2 = np.array([[0, 1], [1, 0], [1, 1], [2, 3]], np.int32)
    g2 = oracle.build_csr(4, uv2)
    d2, _ = oracle.bfs(g2, 0)
    assert oracle.component_tuples(uv2, d2) == 3


def test_sample_roots():
    uv, g = oracle.kron_graph(12, 16, 4)
    r1 = oracle.sample_roots(g, 12, 4, 64)
    r2 = oracle.sample_roots(g, 12, 4, 64)
    assert np.array_equal(r1, r2) and len(r1) == 64
    assert len(set(r1.tolist())) == 64
    deg = g.degree()
    assert np.all(deg[r1] > 0) and r1.min() >= 0 and r1.max() < g.n
    # candidate k is Philox(ctr=(k,0,0,2), key=seed)[0] >> (32 - scale); the first accepted
    # root is the first candidate whose degree is non-zero
    for k in range(64):
        c = int(oracle.philox4x32_10([k, 0, 0, 2], [4, 0])[0]) >> (32 - 12)
        if deg[c] > 0:
            assert r1[0] == c
            break
