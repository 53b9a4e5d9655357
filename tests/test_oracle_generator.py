"""Pins for the oracle's Philox4x32-10 and Kronecker generator (oracle/oracle.c).

Each check is fixed by something other than the oracle itself: published
known-answer vectors, the SPEC's stated properties, closed-form probabilities
of the Kronecker initiator, and a chi-square test of
the uniform special case.
"""
import math
import os

import numpy as np
import pytest

import oracle
from tests.graphs import GOLDEN


def _kat_rows():
    rows = []
    with open(os.path.join(GOLDEN, "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            w = [int(x, 16) for x in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,want", _kat_rows())
def test_philox_known_answers(ctr, key, want):
    assert list(oracle.philox4x32_10(ctr, key)) == want


def test_generator_cardinality_and_range():
    # S:104 post: exactly edgefactor * 2^scale pairs ("Scale30 [1B V, 16B E]").
    # S:107's "(scale=1, edgefactor=1) -> exactly 1 pair" contradicts S:104 (1 * 2^1 = 2);
    # DESIGN.md reading R20 follows S:104 and the paper.
    uv = oracle.kron_edges(1, 1, 42)
    assert uv.shape == (2, 2) and set(uv.ravel().tolist()) <= {0, 1}
    uv = oracle.kron_edges(10, 16, 7)
    assert uv.shape == (16 << 10, 2)
    assert uv.min() >= 0 and uv.max() < 1 << 10


def test_generator_determinism_and_ranges():
    # same spec twice -> identical; S:121 edge i depends only on (seed, i)
    a = oracle.kron_edges(10, 16, 7)
    b = oracle.kron_edges(10, 16, 7)
    assert np.array_equal(a, b)
    part = oracle.kron_edges(10, 16, 7, first=1000, count=500)
    assert np.array_equal(part, a[1000:1500])
    c = oracle.kron_edges(10, 16, 8)
    assert not np.array_equal(a, c)


@pytest.mark.parametrize("scale", [1, 2, 5, 8, 12, 16])
def test_scramble_is_a_bijection(scale):
    keys = oracle.scramble_keys(12345)
    img = [oracle.scramble(scale, keys, v) for v in range(1 << scale)]
    assert sorted(img) == list(range(1 << scale))


def test_initiator_bit_frequencies():
    """Before the scramble every level is an independent draw from the initiator:
    P(u bit = 1) = c + d = 0.24, P(v bit = 1) = b + d = 0.24, P(both) = d = 0.05,
    so the observed frequencies must sit within 5 sigma of those closed forms."""
    s = 16
    uv = oracle.kron_edges(s, 16, 3, scramble_labels=False).astype(np.int64)
    M = uv.shape[0]
    for l in range(s):
        ub = (uv[:, 0] >> l) & 1
        vb = (uv[:, 1] >> l) & 1
        for obs, p in ((ub.mean(), 0.24), (vb.mean(), 0.24), ((ub & vb).mean(), 0.05),
                       (((1 - ub) & (1 - vb)).mean(), 0.57)):
            sigma = math.sqrt(p * (1 - p) / M)
            assert abs(obs - p) < 5 * sigma, (l, obs, p)


def test_hub_degree_closed_form():
    """The pre-scramble label 0 is hit by an endpoint with probability 0.76**s per
    endpoint, so its raw arc count has mean 2*M*0.76**s and sd ~ sqrt(mean)."""
    s, ef, seed = 16, 16, 1
    M = ef << s
    uv = oracle.kron_edges(s, ef, seed).astype(np.int64)
    hub = oracle.scramble(s, oracle.scramble_keys(seed), 0)
    raw = int((uv[:, 0] == hub).sum() + (uv[:, 1] == hub).sum())
    mean = 2 * M * 0.76 ** s
    assert abs(raw - mean) < 5 * math.sqrt(mean), (raw, mean)
    deg = np.bincount(uv.ravel(), minlength=1 << s)
    assert deg.argmax() == hub


def test_isolated_fraction_closed_form():
    """A vertex whose pre-scramble label has popcount w is touched by one tuple
    with probability t_w = 2 q_w - r_w, q_w = .76^(s-w) .24^w, r_w = .57^(s-w) .05^w,
    so E[#isolated] = sum_w C(s,w) (1 - t_w)^M."""
    s, ef = 16, 16
    M = ef << s
    uv = oracle.kron_edges(s, ef, 1)
    deg = np.bincount(uv.ravel().astype(np.int64), minlength=1 << s)
    iso = int((deg == 0).sum())
    exp = 0.0
    var = 0.0
    for w in range(s + 1):
        q = 0.76 ** (s - w) * 0.24 ** w
        r = 0.57 ** (s - w) * 0.05 ** w
        p = (1 - (2 * q - r)) ** M
        exp += math.comb(s, w) * p
        var += math.comb(s, w) * p * (1 - p)
    assert abs(iso - exp) < 5 * math.sqrt(var) + 1, (iso, exp)


def test_heavy_tail_spec_example():
    # scale 16, ef 16, seed 1 -> max degree > 100 * median degree
    uv = oracle.kron_edges(16, 16, 1)
    deg = np.bincount(uv.ravel().astype(np.int64), minlength=1 << 16)
    assert deg.max() > 100 * np.median(deg)


def test_uniform_special_case_chi_square():
    """A = B = C = D = 1/4 makes every bit a fair coin, i.e. endpoints uniform on
    [0, 2^s): a chi-square over the 2^s bins must be within 5 sd of its dof."""
    s = 10
    uv = oracle.kron_edges(s, 64, 9, abc=oracle.ER_ABC)
    for col in (0, 1):
        cnt = np.bincount(uv[:, col].astype(np.int64), minlength=1 << s)
        e = uv.shape[0] / (1 << s)
        chi2 = float(((cnt - e) ** 2 / e).sum())
        dof = (1 << s) - 1
        assert abs(chi2 - dof) < 5 * math.sqrt(2 * dof), chi2


def _rank(x):
    r = np.empty(len(x))
    r[np.argsort(x, kind="stable")] = np.arange(len(x))
    return r


@pytest.mark.parametrize("seed", [1, 2, 7])
def test_scramble_randomly_permutes_labels(seed):
    """S:104 "vertex labels are randomly permuted after generation": besides being a
    bijection (above) the scramble must look like a random permutation.  A uniform
    random permutation of n labels has Poisson(1) fixed points and a Spearman rank
    correlation with the identity of sd 1/sqrt(n-1); the pre-scramble popcount (which
    fixes a vertex's expected degree, SURVEY c1 v') must not predict the new label.
    An identity or order-preserving "scramble" fails every one of these."""
    s = 16
    n = 1 << s
    keys = oracle.scramble_keys(seed)
    v = np.arange(n)
    img = np.array([oracle.scramble(s, keys, int(x)) for x in v], np.int64)
    assert img[0] != 0
    assert int((img == v).sum()) <= 8                      # P(Poisson(1) > 8) < 1e-6
    sd = 1 / math.sqrt(n - 1)
    rho = np.corrcoef(_rank(v), _rank(img))[0, 1]
    assert abs(rho) < 5 * sd, rho
    pop = np.array([bin(x).count("1") for x in range(n)], np.float64)
    r_pop = np.corrcoef(pop, img.astype(np.float64))[0, 1]
    assert abs(r_pop) < 5 * sd, r_pop
    # the 17 highest-expected-degree labels (popcount <= 1) land anywhere: their mean
    # new label is within 5 sd of (n-1)/2 (sd of a mean of k uniform draws)
    top = img[pop <= 1].astype(np.float64)
    assert abs(top.mean() - (n - 1) / 2) < 5 * (n / math.sqrt(12 * len(top))), top.mean()

