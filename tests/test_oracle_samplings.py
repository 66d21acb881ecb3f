"""Pins for the oracle's other doubly uniform samplings.

tau-independent, (tau, p_b)-binomial (PAPER.md:448-456,
exponent reading R13), general doubly uniform DU(q) (eq:p(S))
and the ESO constant of thm:ESO-DU (tbl:ESO :339-350).
Checked against: the paper's own q_k recursion and printed q-values, the
moments the paper prints, exhaustive subset laws on tiny n (doubly uniform:
P(S) depends only on |S|), exact ESO by enumeration incl. the DSO tightness
matrix (equality), and a bit-exact pure-Python twin (oracle/ref_sampler.py).
"""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
from scipy import stats

from oracle import ref_sampler
from paper_1212_0873_b200 import instances as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def paper_independent_q(n, tau):
    """q_k of the tau-independent sampling exactly as PAPER.md:440-444 defines it:
    q_k = C(n,k) c_k, c_1 = (1/n)^tau, c_k = (k/n)^tau - sum_{i<k} C(k,i) c_i."""
    c = {}
    for k in range(1, tau + 1):
        c[k] = Fraction(k, n) ** tau - sum(math.comb(k, i) * c[i] for i in range(1, k))
    return {k: math.comb(n, k) * c[k] for k in range(1, tau + 1)}


def sizes(slots):
    return int(np.sum(np.asarray(slots) >= 0))


# ------------------------------------------------------------ tau-independent
def test_independent_law_recursion_matches_printed_q():
    g = json.load(open(os.path.join(GOLDEN, "paper_values.json")))["tau_independent_q"]
    q = paper_independent_q(g["n"], g["tau"])
    for k, want in g["q"].items():
        assert round(float(q[int(k)]), 4) == want
    assert sum(q.values()) == 1


@pytest.mark.parametrize("n,tau", [(1, 1), (5, 3), (12, 7), (30, 30), (1000, 8), (200, 40)])
def test_independent_moments_closed_form_vs_recursion(orc, n, tau):
    q = paper_independent_q(n, tau)
    e1 = sum(k * v for k, v in q.items())
    e2 = sum(k * k * v for k, v in q.items())
    m1, m2 = orc.moments(orc.Sampling("independent", tau), n)
    assert m1 == pytest.approx(float(e1), rel=1e-11)
    assert m2 == pytest.approx(float(e2), rel=1e-11)


def test_independent_sampler_cardinality_law(orc):
    n, tau, N = 1000, 8, 30000
    S = orc.Sampling("independent", tau)
    card = np.bincount([sizes(orc.sample_kind(S, 3, k, n)) for k in range(N)], minlength=tau + 1)
    q = paper_independent_q(n, tau)
    for k in (6, 7, 8):
        p = float(q[k])
        sd = math.sqrt(max(p, 1e-4) * (1 - p) / N)
        assert abs(card[k] / N - p) < 5 * sd + 5e-5


def test_independent_twin_and_processor_semantics(orc):
    for n, tau in ((7, 5), (50, 20), (3, 3), (1000, 64)):
        S = orc.Sampling("independent", tau)
        for k in range(15):
            got = orc.sample_kind(S, 11, k, n)
            assert list(got) == ref_sampler.sample_independent(11, k, tau, n)
            act = got[got >= 0]
            assert len(set(act.tolist())) == len(act)           # each block updated once
            # processor j picks its own first accepted draw; the lowest j keeps a shared pick
            picks = [orc.draw(11, k, 0, j, 3, n) for j in range(tau)]
            for j in range(tau):
                assert got[j] == (picks[j] if picks[j] not in picks[:j] else -1)


# ------------------------------------------------------------ binomial
def test_binomial_moments_printed_and_beta_row(orc):
    # E|S| = tau p_b, E|S|^2 = tau p_b (1 + tau p_b - p_b); tbl:ESO row
    for tau, pb, n, om in ((16, 0.3, 100, 7), (1, 0.9, 10, 3), (50, 1.0, 50, 12)):
        S = orc.Sampling("binomial", tau, p_b=pb)
        e1, e2 = orc.moments(S, n)
        assert e1 == pytest.approx(tau * pb) and e2 == pytest.approx(tau * pb * (1 + tau * pb - pb))
        assert orc.beta_sampling(om, n, S) == pytest.approx(1 + pb * (om - 1) * (tau - 1) / max(1, n - 1))
    # p_b = 1 is the tau-nice sampling, beta included
    assert orc.beta_sampling(9, 40, orc.Sampling("binomial", 12, p_b=1.0)) == pytest.approx(orc.beta(9, 12, 40))


def test_binomial_sampler_law_and_twin(orc):
    n, tau, pb, N = 40, 12, 0.35, 20000
    S = orc.Sampling("binomial", tau, p_b=pb)
    card = np.bincount([sizes(orc.sample_kind(S, 5, k, n)) for k in range(N)], minlength=tau + 1)
    # reading R13: q_k = C(tau,k) p_b^k (1-p_b)^(tau-k)
    want = np.array([math.comb(tau, k) * pb ** k * (1 - pb) ** (tau - k) for k in range(tau + 1)])
    keep = want * N >= 5
    chi = np.sum((card[keep] - N * want[keep]) ** 2 / (N * want[keep]))
    assert stats.chi2.sf(chi, keep.sum() - 1) > 1e-3
    for k in range(20):
        assert list(orc.sample_kind(S, 5, k, n)) == ref_sampler.sample_binomial(5, k, tau, n, pb)
    nice = orc.Sampling("binomial", tau, p_b=1.0)
    for k in range(10):
        assert np.array_equal(orc.sample_kind(nice, 5, k, n), orc.sample(5, k, tau, n))


# ------------------------------------------------------------ general DU(q)
def test_du_sampler_size_law_twin_and_special_cases(orc):
    n, tau = 30, 6
    q = np.array([0.05, 0.1, 0.0, 0.3, 0.25, 0.1, 0.2])
    S = orc.Sampling("du", tau, q=q)
    N = 20000
    card = np.bincount([sizes(orc.sample_kind(S, 8, k, n)) for k in range(N)], minlength=tau + 1)
    keep = q > 0
    chi = np.sum((card[keep] - N * q[keep]) ** 2 / (N * q[keep]))
    assert stats.chi2.sf(chi, keep.sum() - 1) > 1e-3
    assert card[2] == 0
    for k in range(20):
        assert list(orc.sample_kind(S, 8, k, n)) == ref_sampler.sample_du(8, k, tau, n, q)
    e1, e2 = orc.moments(S, n)
    assert e1 == pytest.approx(np.dot(np.arange(tau + 1), q)) and e2 == pytest.approx(np.dot(np.arange(tau + 1) ** 2, q))
    # q = e_tau: tau-nice; q = e_1: serial (beta = 1, tbl:ESO serial row)
    e_tau = np.zeros(tau + 1)
    e_tau[tau] = 1
    for k in range(10):
        assert np.array_equal(orc.sample_kind(orc.Sampling("du", tau, q=e_tau), 8, k, n), orc.sample(8, k, tau, n))
    e_1 = np.zeros(tau + 1)
    e_1[1] = 1
    assert orc.beta_sampling(5, n, orc.Sampling("du", tau, q=e_1)) == 1.0
    assert orc.beta_sampling(5, n, orc.Sampling("du", tau, q=e_tau)) == pytest.approx(orc.beta(5, tau, n))


@pytest.mark.parametrize("kind", ["independent", "binomial", "du"])
def test_doubly_uniform_exhaustive(orc, kind):
    # DU: P(S) = q_|S| / C(n,|S|) -- uniform within every size
    n, tau, N = 6, 3, 60000
    S = {"independent": orc.Sampling("independent", tau), "binomial": orc.Sampling("binomial", tau, p_b=0.6),
         "du": orc.Sampling("du", tau, q=[0.1, 0.2, 0.3, 0.4])}[kind]
    counts = {}
    for k in range(N):
        s = orc.sample_kind(S, 21, k, n)
        key = tuple(sorted(int(v) for v in s if v >= 0))
        counts[key] = counts.get(key, 0) + 1
    for size in range(1, tau + 1):
        subsets = list(itertools.combinations(range(n), size))
        obs = np.array([counts.get(sub, 0) for sub in subsets])
        if obs.sum() < 50:
            continue
        chi = np.sum((obs - obs.mean()) ** 2 / obs.mean())
        assert stats.chi2.sf(chi, len(subsets) - 1) > 1e-4, (kind, size)


# ------------------------------------------------------------ ESO for DU samplings
def _law(orc, S, n):
    """P(|S| = k), k = 0..tau, of each sampling, from its definition (not from the sampler)."""
    tau = S.tau
    if S.kind == "independent":
        q = paper_independent_q(n, tau)
        return np.array([0.0] + [float(q[k]) for k in range(1, tau + 1)])
    if S.kind == "binomial":
        return np.array([math.comb(tau, k) * S.p_b ** k * (1 - S.p_b) ** (tau - k) for k in range(tau + 1)])
    return np.asarray(S.q, dtype=np.float64)


@pytest.mark.parametrize("S_args", [("independent", 3, 1.0, None), ("binomial", 4, 0.4, None),
                                    ("du", 4, 1.0, [0.0, 0.3, 0.1, 0.2, 0.4])])
def test_eso_du_by_exact_enumeration(orc, S_args):
    # thm:ESO-DU: E f(x + h_[S]) <= f(x) + E|S|/n (<grad f, h> + beta/2 ||h||_L^2), f = 1/2||Ax-b||^2,
    # exact expectation with P(S) = q_|S| / C(n,|S|); equality on the DSO tightness matrix (h ~ 1)
    kind, tau, pb, q = S_args
    S = orc.Sampling(kind, tau, p_b=pb, q=q)
    rng = np.random.default_rng(4)
    for trial in range(8):
        m, n = 9, 6
        lens = rng.integers(1, m + 1, size=n)
        colptr, rowidx, val = I.random_csc(m, n, lens, seed=200 + trial)
        c, r, v = colptr.numpy(), rowidx.numpy(), val.numpy()
        A = np.zeros((m, n))
        for i in range(n):
            A[r[c[i]:c[i + 1]], i] = v[c[i]:c[i + 1]]
        b = rng.normal(size=m)
        om = orc.omega(m, r)
        beta = orc.beta_sampling(om, n, S)
        L = (A ** 2).sum(0)
        law = _law(orc, S, n)
        f = lambda z: 0.5 * np.sum((A @ z - b) ** 2)
        x, h = rng.normal(size=n), rng.normal(size=n)
        grad = A.T @ (A @ x - b)
        Ef = 0.0
        for size in range(tau + 1):
            subs = list(itertools.combinations(range(n), size))
            for sub in subs:
                y = x.copy()
                y[list(sub)] += h[list(sub)]
                Ef += law[size] / len(subs) * f(y)
        e1 = float(np.dot(np.arange(tau + 1), law))
        bound = f(x) + e1 / n * (grad @ h + 0.5 * beta * np.sum(L * h * h))
        assert Ef <= bound + 1e-10
    colptr, rowidx, val = I.equal_row_01_matrix(12, 8, 4, seed=1)
    c, r, v = colptr.numpy(), rowidx.numpy(), val.numpy()
    m, n = 12, 8
    A = np.zeros((m, n))
    for i in range(n):
        A[r[c[i]:c[i + 1]], i] = v[c[i]:c[i + 1]]
    S8 = orc.Sampling(kind, tau, p_b=pb, q=q)
    beta = orc.beta_sampling(orc.omega(m, r), n, S8)
    law = _law(orc, S8, n)
    L = (A ** 2).sum(0)
    h = np.ones(n) / math.sqrt(L[0])
    f = lambda z: 0.5 * np.sum((A @ z) ** 2)
    Ef = 0.0
    for size in range(tau + 1):
        subs = list(itertools.combinations(range(n), size))
        for sub in subs:
            Ef += law[size] / len(subs) * f(np.where(np.isin(np.arange(n), sub), h, 0.0))
    e1 = float(np.dot(np.arange(tau + 1), law))
    assert Ef == pytest.approx(e1 / n * 0.5 * beta * np.sum(L * h * h), rel=1e-10)


# ------------------------------------------------------------ runs
def test_runs_with_du_samplings(orc):
    m, n = 60, 40
    colptr, rowidx, val = I.random_csc(m, n, np.full(n, 5), seed=3)
    b = I.random_b(m, seed=3)
    c, r, v, bb = colptr.numpy(), rowidx.numpy(), val.numpy(), b.numpy()
    lam = I.lam_for(colptr, rowidx, val, b)
    F0 = orc.objective(m, c, r, v, bb, lam, np.zeros(n))
    Fstar = orc.objective(m, c, r, v, bb, lam, orc.run(m, c, r, v, bb, lam, n, 3000, seed=1).x)
    for S in (orc.Sampling("independent", 10), orc.Sampling("binomial", 10, p_b=0.5),
              orc.Sampling("du", 10, q=np.full(11, 1 / 11))):
        res = orc.run(m, c, r, v, bb, lam, S.tau, 400, seed=2, sampling=S, keep_slots=True)
        assert res.beta == pytest.approx(orc.beta_sampling(res.omega, n, S))
        for k in range(5):
            assert np.array_equal(res.slots[k], orc.sample_kind(S, 2, k, n))
        F = orc.objective(m, c, r, v, bb, lam, res.x)
        assert F - Fstar <= 1e-3 * (F0 - Fstar)   # every DU sampling drives F to the same minimum
    # p_b = 1 binomial == nice, bit for bit
    a = orc.run(m, c, r, v, bb, lam, 8, 50, seed=4, sampling=orc.Sampling("binomial", 8, p_b=1.0)).x
    bnice = orc.run(m, c, r, v, bb, lam, 8, 50, seed=4).x
    assert np.array_equal(a, bnice)
