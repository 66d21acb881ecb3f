"""Pins for the oracle's tau-nice sampler.

The paper fixes only the LAW of S_k: tau-nice = uniform over all tau-subsets
of [n].  These tests check the oracle's sampler against
that law and its closed-form moments, against the paper's printed
tau-independent q-values (the law of the round-0 draws), against published
Philox known-answer vectors, and against an independently written pure-Python
twin (oracle/ref_sampler.py).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import ref_sampler

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            w = [int(t, 16) for t in line.split()]
            rows.append((w[0:4], w[4:6], w[6:10]))
    return rows


def test_philox_known_answers(orc):
    # P1 (host half): Random123 KAT vectors, tests/golden/philox4x32_10_kat.txt
    for ctr, key, out in _kat():
        assert list(orc.philox4x32_10(ctr, key)) == out
        assert ref_sampler.philox4x32_10(ctr, key) == out


def test_draw_matches_twin_including_rejections(orc):
    # Lemire map incl. the rejection branch: for n just above 2^63 about half
    # of all 64-bit words are rejected, so both branches are exercised.
    rng = np.random.default_rng(1)
    ns = [1, 2, 3, 1000, 999_999_937, (1 << 31) - 1, (1 << 63) + 12345, (1 << 64) - 5]
    rejected = 0
    for n in ns:
        for _ in range(200):
            seed = int(rng.integers(0, 1 << 63)) * 2 + 1
            k, rho, j, tag = (int(v) for v in rng.integers(0, 1 << 32, size=4))
            a = orc.draw(seed, k, rho, j, tag, n)
            b = ref_sampler.draw(seed, k, rho, j, tag, n)
            assert a == b
            if a is None:
                rejected += 1
            else:
                assert 0 <= a < n
    assert rejected > 50


@pytest.mark.parametrize("n,tau", [(1, 1), (2, 1), (2, 2), (5, 2), (7, 5), (20, 8), (20, 15),
                                   (100, 50), (100, 51), (97, 96), (1000, 32), (64, 64)])
def test_sampler_twin_bitexact(orc, n, tau):
    # P2(v): C oracle == independent pure-Python twin, slot order included
    for seed in (0, 1, 0xDEADBEEFCAFE):
        for k in (0, 1, 17, 4_000_000_000):
            a = orc.sample(seed, k, tau, n)
            b = ref_sampler.sample(seed, k, tau, n)
            assert list(a) == list(b)
            assert len(set(a.tolist())) == tau
            assert a.min() >= 0 and a.max() < n


def test_tau_equals_n_is_fully_parallel(orc):
    # P2(iv): tau = n gives [n] (fully parallel sampling)
    for n in (1, 2, 9, 128):
        assert orc.sample(3, 5, n, n).tolist() == list(range(n))


def test_serial_sampling_uniform(orc):
    # P2(iv): tau = 1 -> uniform singletons (serial sampling)
    n, N = 7, 14000
    counts = np.zeros(n)
    for k in range(N):
        s = orc.sample(11, k, 1, n)
        counts[s[0]] += 1
    p = stats.chisquare(counts).pvalue
    assert p > 1e-4


@pytest.mark.parametrize("n,tau,N", [(6, 3, 12000), (7, 5, 10500), (5, 2, 8000)])
def test_exhaustive_subset_law(orc, n, tau, N):
    # P2(i): P(S) = 1/C(n,tau) for every tau-subset (tau-nice, PAPER.md:436 with eq:p(S) :422)
    subsets = {s: 0 for s in itertools.combinations(range(n), tau)}
    for k in range(N):
        s = tuple(sorted(orc.sample(2024, k, tau, n).tolist()))
        subsets[s] += 1
    counts = np.array(list(subsets.values()), dtype=float)
    assert counts.min() > 0
    assert stats.chisquare(counts).pvalue > 1e-4


def test_element_and_pair_probabilities(orc):
    # P2(ii): p_i = tau/n (eq:simple2unif PAPER.md:543) and
    # p_ij = E[|S|^2-|S|]/(n(n-1)) = tau(tau-1)/(n(n-1)) (eq:p_ij_equals PAPER.md:552)
    n, tau, N = 40, 9, 20000
    inc = np.zeros((N, n), dtype=np.float64)
    for k in range(N):
        inc[k, orc.sample(77, k, tau, n)] = 1.0
    pi = inc.mean(0)
    p = tau / n
    sd = math.sqrt(p * (1 - p) / N)
    assert np.all(np.abs(pi - p) < 5 * sd)
    pij = (inc.T @ inc) / N
    off = pij[~np.eye(n, dtype=bool)]
    q = tau * (tau - 1) / (n * (n - 1))
    sdq = math.sqrt(q * (1 - q) / N)
    assert abs(off.mean() - q) < 5 * sdq / math.sqrt(n)  # mean over pairs: much tighter
    assert np.all(np.abs(off - q) < 6 * sdq)


def test_intersection_second_moment(orc):
    # eq:00sjs738: E|J cap S|^2 = (|J| tau/n)(1 + (|J|-1)(tau-1)/max(1,n-1))
    n, tau, N = 30, 7, 20000
    J = np.array([0, 3, 4, 17, 29])
    vals = np.empty(N)
    for k in range(N):
        s = orc.sample(5, k, tau, n)
        vals[k] = np.isin(s, J).sum()
    want = len(J) * tau / n * (1 + (len(J) - 1) * (tau - 1) / max(1, n - 1))
    got = (vals ** 2).mean()
    se = (vals ** 2).std() / math.sqrt(N)
    assert abs(got - want) < 5 * se


def test_round0_draws_follow_paper_tau_independent_law(orc):
    # P2(iii): round-0 draws are tau iid uniform picks, i.e. the tau-independent
    # sampling of PAPER.md:440-446, whose cardinality law the paper prints for
    # n=1000, tau=8: q8=0.9723, q7=0.0274, q6=0.0003 (tests/golden/paper_values.json).
    g = json.load(open(os.path.join(GOLDEN, "paper_values.json")))["tau_independent_q"]
    n, tau = g["n"], g["tau"]
    N = 40000
    card = np.zeros(tau + 1)
    for k in range(N):
        vals = {orc.draw(99, k, 0, j, 1, n) for j in range(tau)}
        card[len(vals)] += 1
    freq = card / N
    for kk, q in g["q"].items():
        kk = int(kk)
        sd = math.sqrt(max(q, 1e-4) * (1 - q) / N)
        assert abs(freq[kk] - q) < 5 * sd + 5e-5, (kk, freq[kk], q)
    # closed form of the paper's recursion at tau=8: q8 = prod_{j<8} (1 - j/n)
    q8 = np.prod([1 - j / n for j in range(tau)])
    assert round(q8, 4) == g["q"]["8"]
