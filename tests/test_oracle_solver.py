"""Pins for the oracle's PCDM1/LASSO arithmetic.

Each test checks the oracle against something the paper or plain mathematics
fixes -- brute force on dense matrices, closed forms, paper-printed values,
the ESO identities, KKT optimality and exact LASSO solutions -- never against
a retyped copy of its own formula.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch
from scipy import optimize

from paper_1212_0873_b200 import instances as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def dense(m, colptr, rowidx, val):
    A = np.zeros((m, len(colptr) - 1))
    for i in range(len(colptr) - 1):
        for p in range(colptr[i], colptr[i + 1]):
            A[rowidx[p], i] = val[p]
    return A


def small_problem(m, n, lens, seed=0, lam_frac=0.1):
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=seed)
    b = I.random_b(m, seed=seed)
    lam = I.lam_for(colptr, rowidx, val, b, lam_frac)
    return (colptr.numpy(), rowidx.numpy(), val.numpy(), b.numpy(), lam)


def F_dense(A, b, lam, x):
    r = A @ x - b.astype(np.float64)
    return 0.5 * r @ r + lam * np.abs(x).sum()


def soft(u, t):
    return np.sign(u) * np.maximum(np.abs(u) - t, 0.0)


# ---------------------------------------------------------------- P3: omega
def test_omega_brute_force(orc):
    rng = np.random.default_rng(0)
    for trial in range(30):
        m, n = int(rng.integers(1, 40)), int(rng.integers(1, 30))
        lens = rng.integers(0, m + 1, size=n)
        c, r, v, b, lam = small_problem(m, n, lens, seed=trial)
        A = dense(m, c, r, v)
        want = int((A != 0).sum(1).max()) if A.size else 0
        # stored entries == nonzeros here (N(0,1) values are never exactly 0)
        assert orc.omega(m, r) == want


def test_omega_special_matrices(orc):
    # diagonal -> 1 ; one fully dense row over n columns -> n (SPEC.md:50-51 examples)
    n = 9
    assert orc.omega(n, np.arange(n, dtype=np.int32)) == 1
    assert orc.omega(3, np.ones(n, dtype=np.int32)) == n


# ---------------------------------------------------------------- P4: beta
def test_beta_special_cases(orc):
    # tbl:ESO: tau=1 -> 1 (serial), tau=n -> omega (fully
    # parallel); omega=1 -> 1 for every tau (separable)
    for n, om in [(10, 3), (1000, 35), (7, 7)]:
        assert orc.beta(om, 1, n) == 1.0
        assert orc.beta(om, n, n) == pytest.approx(om, rel=1e-15)
        for tau in (1, 2, n):
            assert orc.beta(1, tau, n) == 1.0
    assert orc.beta(5, 1, 1) == 1.0  # n = 1: max(1, n-1) reading R#4


def test_beta_paper_values(orc):
    g = json.load(open(os.path.join(GOLDEN, "paper_values.json")))
    rc = g["rcv1_beta"]
    b = orc.beta(rc["omega"], rc["tau"], rc["n"])
    assert round(b, 2) == rc["beta"]           # "beta = 7.46"
    assert round(rc["tau"] / b, 2) == rc["psf"]  # "PSF = tau/beta = 2.15"
    bl = g["billion_lasso"]
    for tau in bl["taus"]:
        assert orc.beta(bl["omega"], tau, bl["n"]) - 1.0 < 1e-6


# ---------------------------------------------------------------- P5: prox
def test_prox_paper_example(orc):
    g = json.load(open(os.path.join(GOLDEN, "paper_values.json")))["soft_threshold_example"]
    xp = orc.prox(g["x"], g["g"], g["s"], g["lam"])
    assert xp - g["x"] == g["h"]


def test_prox_vs_brute_force_minimisation(orc):
    # h_i = argmin_t g t + (s/2) t^2 + lam |x + t|  (eq:h(x) block form)
    rng = np.random.default_rng(3)
    for _ in range(300):
        x, g = rng.normal(scale=2, size=2)
        s = float(rng.uniform(0.1, 5))
        lam = float(rng.choice([0.0, rng.uniform(0, 3)]))
        phi = lambda t: g * t + 0.5 * s * t * t + lam * np.abs(x + t)
        R = (abs(g) + lam) / s + abs(x) + 1.0
        grid = np.linspace(-R, R, 80001)
        t0 = grid[np.argmin(phi(grid))]
        res = optimize.minimize_scalar(phi, bounds=(t0 - 2 * R / 8e4, t0 + 2 * R / 8e4), method="bounded",
                                       options={"xatol": 1e-12})
        tbest = res.x if phi(res.x) <= phi(t0) else t0
        # the kink t = -x is a candidate minimiser the smooth search can miss
        if phi(-x) <= phi(tbest):
            tbest = -x
        h = orc.prox(x, g, s, lam) - x
        assert phi(h) <= phi(tbest) + 1e-12
        assert abs(h - tbest) < 1e-6


def test_prox_lambda_zero_and_ties(orc):
    assert orc.prox(1.0, 4.0, 2.0, 0.0) == pytest.approx(1.0 - 2.0)  # h = -g/s
    # |u| == lam/s exactly -> 0 (reading R#6)
    assert orc.prox(0.0, -1.0, 2.0, 1.0) == 0.0
    # empty column (s=0, reading R#5)
    assert orc.prox(0.7, 0.0, 0.0, 1.0) == 0.0
    assert orc.prox(0.7, 0.0, 0.0, 0.0) == 0.7


# ------------------------------------------------- L, residual, objective vs dense
def test_col_norms_residual_objective_dense(orc):
    m, n = 30, 12
    c, r, v, b, lam = small_problem(m, n, [0, 1, 5, 30, 3, 3, 7, 2, 9, 10, 1, 4])
    A = dense(m, c, r, v)
    np.testing.assert_allclose(orc.col_norms(c, v), (A ** 2).sum(0), rtol=1e-15)
    x = np.random.default_rng(1).normal(size=n)
    x[[1, 4]] = 0.0
    np.testing.assert_allclose(orc.residual(m, c, r, v, b, x), A @ x - b, rtol=1e-12, atol=1e-12)
    assert orc.objective(m, c, r, v, b, lam, x) == pytest.approx(F_dense(A, b, lam, x), rel=1e-13)


# ------------------------------------- P11: one iteration == dense definition
@pytest.mark.parametrize("tau", [1, 3, 8, 20])
def test_one_iteration_equals_dense_definition(orc, tau):
    # x_{k+1} = x_k + (h(x_k))_[S_k]  (alg:PCD1 step 4; h from
    # eq:h(x), eq:H_{beta,w} with w = L, Omega = lam||.||_1), computed densely:
    # grad f = A^T (A x - b); h_i = soft(x_i - grad_i/(beta L_i), lam/(beta L_i)) - x_i
    m, n = 25, 20
    lens = np.random.default_rng(tau).integers(1, 8, size=n)
    c, r, v, b, lam = small_problem(m, n, lens, seed=tau)
    A = dense(m, c, r, v)
    x0 = np.random.default_rng(5).normal(size=n)
    x0[::3] = 0.0
    for first in (0, 7):
        res = orc.run(m, c, r, v, b, lam, tau, 1, seed=42, x0=x0, first_iter=first)
        S = orc.sample(42, first, tau, n)
        L = (A ** 2).sum(0)
        om = int((A != 0).sum(1).max())
        beta = 1 + (om - 1) * (tau - 1) / max(1, n - 1)
        grad = A.T @ (A @ x0 - b)
        want = x0.copy()
        for i in S:
            s = beta * L[i]
            want[i] = soft(x0[i] - grad[i] / s, lam / s)
        np.testing.assert_allclose(res.x, want, rtol=1e-12, atol=1e-13)


# --------------------------------------------------- P12: residual bookkeeping
def test_maintained_residual_matches_recomputed(orc):
    m, n = 60, 50
    c, r, v, b, lam = small_problem(m, n, np.full(n, 6), seed=9)
    A = dense(m, c, r, v)
    res = orc.run(m, c, r, v, b, lam, 7, 3000, seed=1, refresh_every=-1)
    exact = A @ res.x - b
    assert np.max(np.abs(res.r - exact)) <= 1e-12 * max(1.0, np.max(np.abs(exact)))
    # refresh cadence is a rounding-only change in fp64 (O8)
    res2 = orc.run(m, c, r, v, b, lam, 7, 3000, seed=1, refresh_every=1)
    np.testing.assert_allclose(res2.x, res.x, rtol=1e-9, atol=1e-12)


# ------------------------------------------------------ P6: tau = 1 serial CDM
def test_serial_steps_are_exact_coordinate_minimisers(orc):
    # tbl:special_cases: P(|S|=1)=1 gives serial random CDM; beta=1
    # and f is exactly quadratic along e_i with curvature L_i, so each step
    # minimises F along that coordinate and F never increases.
    m, n = 30, 15
    c, r, v, b, lam = small_problem(m, n, np.full(n, 5), seed=2)
    A = dense(m, c, r, v)
    x = np.zeros(n)
    Fprev = F_dense(A, b, lam, x)
    for k in range(60):
        res = orc.run(m, c, r, v, b, lam, 1, 1, seed=8, x0=x, first_iter=k)
        i = int(orc.sample(8, k, 1, n)[0])
        d = res.x[i] - x[i]
        for t in np.linspace(d - 2, d + 2, 81):
            y = x.copy()
            y[i] += t
            assert F_dense(A, b, lam, res.x) <= F_dense(A, b, lam, y) + 1e-12
        Fk = F_dense(A, b, lam, res.x)
        assert Fk <= Fprev + 1e-12
        Fprev, x = Fk, res.x


# --------------------------------------------------- P8: tau = n monotonic
def test_fully_parallel_is_monotone(orc):
    # tbl:ESO fully parallel row: beta = omega, ESO monotonic
    m, n = 40, 25
    c, r, v, b, lam = small_problem(m, n, np.random.default_rng(4).integers(1, 10, size=n), seed=4)
    x = np.zeros(n)
    Fs = [orc.objective(m, c, r, v, b, lam, x)]
    for k in range(40):
        x = orc.run(m, c, r, v, b, lam, n, 1, seed=0, x0=x, first_iter=k).x
        Fs.append(orc.objective(m, c, r, v, b, lam, x))
    assert all(Fs[i + 1] <= Fs[i] + 1e-12 for i in range(len(Fs) - 1))
    assert Fs[-1] < Fs[0]


# ----------------------------------------------------- P7: omega = 1 separable
def test_separable_problem_solved_in_one_full_step(orc):
    # omega = 1 (disjoint column supports): beta = 1 for every tau
    # and each coordinate jumps to x_i* = soft(a_i^T b / L_i, lam / L_i) (eq:h(x)
    # with r = -b restricted to column i), so tau = n solves in one iteration.
    n, per = 12, 3
    m = n * per + 5
    perm = np.random.default_rng(0).permutation(m)
    colptr = np.arange(0, n * per + 1, per, dtype=np.int64)
    rowidx = np.concatenate([np.sort(perm[i * per:(i + 1) * per]) for i in range(n)]).astype(np.int32)
    val = np.random.default_rng(1).normal(size=n * per).astype(np.float32)
    b = np.random.default_rng(2).normal(size=m).astype(np.float32)
    A = dense(m, colptr, rowidx, val)
    lam = 0.3
    assert orc.omega(m, rowidx) == 1
    res = orc.run(m, colptr, rowidx, val, b, lam, n, 1, seed=3)
    L = (A ** 2).sum(0)
    xstar = soft(A.T @ b / L, lam / L)
    np.testing.assert_allclose(res.x, xstar, rtol=1e-12, atol=1e-14)
    Fstar = 0.5 * np.sum((A @ xstar - b) ** 2) + lam * np.abs(xstar).sum()
    assert orc.objective(m, colptr, rowidx, val, b, lam, res.x) == pytest.approx(Fstar, rel=1e-12)
    # and it stays there
    res2 = orc.run(m, colptr, rowidx, val, b, lam, 5, 50, seed=3, x0=res.x)
    np.testing.assert_allclose(res2.x, xstar, rtol=1e-12, atol=1e-14)


# ----------------------------------------------------------- P9: ESO / eq:1
def _h_full(orc, m, c, r, v, b, lam, x, beta):
    """h(x) for all blocks = one fully parallel step taken with the given beta."""
    n = len(c) - 1
    return orc.run(m, c, r, v, b, lam, n, 1, seed=0, x0=x, beta_override=beta).x - x


def test_expected_decrease_eq1_exact_enumeration(orc):
    # eq:1: E F(x + h_[S]) <= (1-tau/n) F(x) + (tau/n) H_{beta,L}(x,h) <= F(x)
    m, n, tau = 14, 8, 3
    c, r, v, b, lam = small_problem(m, n, [3, 4, 2, 5, 3, 1, 4, 2], seed=11)
    A = dense(m, c, r, v)
    L = (A ** 2).sum(0)
    beta = orc.beta(orc.omega(m, r), tau, n)
    x = np.random.default_rng(2).normal(size=n)
    h = _h_full(orc, m, c, r, v, b, lam, x, beta)
    Fx = F_dense(A, b, lam, x)
    grad = A.T @ (A @ x - b)
    H = 0.5 * np.sum((A @ x - b) ** 2) + grad @ h + 0.5 * beta * np.sum(L * h * h) \
        + lam * np.abs(x + h).sum()
    vals = []
    for S in itertools.combinations(range(n), tau):
        y = x.copy()
        y[list(S)] += h[list(S)]
        vals.append(F_dense(A, b, lam, y))
    EF = np.mean(vals)
    a = tau / n
    assert EF <= (1 - a) * Fx + a * H + 1e-12
    assert (1 - a) * Fx + a * H <= Fx + 1e-12


def test_expected_one_step_monte_carlo(orc):
    # P9(i): mean over seeds of one oracle step == exact expectation over all tau-subsets
    m, n, tau = 14, 8, 3
    c, r, v, b, lam = small_problem(m, n, [3, 4, 2, 5, 3, 1, 4, 2], seed=12)
    A = dense(m, c, r, v)
    x = np.random.default_rng(3).normal(size=n)
    beta = orc.beta(orc.omega(m, r), tau, n)
    h = _h_full(orc, m, c, r, v, b, lam, x, beta)
    exact = []
    for S in itertools.combinations(range(n), tau):
        y = x.copy()
        y[list(S)] += h[list(S)]
        exact.append(F_dense(A, b, lam, y))
    mc = np.array([orc.objective(m, c, r, v, b, lam,
                                 orc.run(m, c, r, v, b, lam, tau, 1, seed=s, x0=x).x)
                   for s in range(4000)])
    assert abs(mc.mean() - np.mean(exact)) < 5 * mc.std() / math.sqrt(len(mc))


def test_eso_psd_condition_and_tightness(orc):
    # thm:ESO-nice for f = 1/2||Ax||^2 is equivalent to
    # (tau/n)(beta-1) D - p2 (A^T A - D) >= 0 with p2 = tau(tau-1)/(n(n-1)).
    rng = np.random.default_rng(7)
    for trial in range(20):
        m, n = int(rng.integers(3, 12)), int(rng.integers(2, 9))
        lens = rng.integers(1, m + 1, size=n)
        c, r, v, b, lam = small_problem(m, n, lens, seed=100 + trial)
        A = dense(m, c, r, v)
        G = A.T @ A
        D = np.diag(np.diag(G))
        om = orc.omega(m, r)
        for tau in range(1, n + 1):
            beta = orc.beta(om, tau, n)
            p2 = tau * (tau - 1) / (n * max(1, n - 1))
            M = (tau / n) * (beta - 1) * D - p2 * (G - D)
            assert np.linalg.eigvalsh(M).min() >= -1e-9 * max(1.0, np.abs(M).max())
    # P9(iv): DSO tightness construction: 0-1 matrix, omega ones
    # per row, k ones per column, h = k^{-1/2} 1 -> ESO holds with EQUALITY.
    colptr, rowidx, val = I.equal_row_01_matrix(12, 8, 4, seed=1)
    c, r, v = colptr.numpy(), rowidx.numpy(), val.numpy()
    m, n = 12, 8
    A = dense(m, c, r, v)
    om = orc.omega(m, r)
    assert om == 4
    L = orc.col_norms(c, v)
    x = np.zeros(n)
    h = np.ones(n) / math.sqrt(L[0])
    f = lambda z: 0.5 * np.sum((A @ z) ** 2)
    for tau in (1, 2, 3, 5, 8):
        beta = orc.beta(om, tau, n)
        Ef = np.mean([f(x + np.where(np.isin(np.arange(n), S), h, 0.0))
                      for S in itertools.combinations(range(n), tau)])
        bound = f(x) + (tau / n) * (0 + 0.5 * beta * np.sum(L * h * h))
        assert Ef == pytest.approx(bound, rel=1e-12)


# --------------------------------------------------------------- P10: KKT
def test_kkt_at_convergence(orc):
    m, n = 40, 20
    c, r, v, b, lam = small_problem(m, n, np.full(n, 6), seed=21, lam_frac=0.2)
    A = dense(m, c, r, v)
    res = orc.run(m, c, r, v, b, lam, 4, 40000, seed=5)
    g = A.T @ (A @ res.x - b)
    z = res.x == 0
    assert np.all(np.abs(g[z]) <= lam * (1 + 1e-9))
    assert np.all(np.abs(g[~z] + lam * np.sign(res.x[~z])) <= 1e-8 * max(1.0, lam))


def _lasso_exact(A, b, lam):
    """Exact LASSO minimiser by sign-pattern enumeration (3^n candidate systems)."""
    n = A.shape[1]
    G, c = A.T @ A, A.T @ b
    best, bestF = None, np.inf
    for signs in itertools.product((-1, 0, 1), repeat=n):
        sg = np.array(signs, dtype=float)
        act = sg != 0
        x = np.zeros(n)
        if act.any():
            try:
                x[act] = np.linalg.solve(G[np.ix_(act, act)], c[act] - lam * sg[act])
            except np.linalg.LinAlgError:
                continue
            if np.any(np.sign(x[act]) != sg[act]):
                continue
        Fv = 0.5 * np.sum((A @ x - b) ** 2) + lam * np.abs(x).sum()
        if Fv < bestF:
            best, bestF = x, Fv
    return best, bestF


def test_converges_to_exact_lasso_solution(orc):
    m, n = 16, 7
    c, r, v, b, lam = small_problem(m, n, np.full(n, 6), seed=31, lam_frac=0.15)
    A = dense(m, c, r, v)
    xstar, Fstar = _lasso_exact(A, b.astype(np.float64), lam)
    for tau in (1, 3, 7):
        res = orc.run(m, c, r, v, b, lam, tau, 30000 // tau, seed=tau)
        assert np.linalg.norm(res.x - xstar) <= 1e-8 * max(1.0, np.linalg.norm(xstar))
        assert orc.objective(m, c, r, v, b, lam, res.x) == pytest.approx(Fstar, rel=1e-12)


# --------------------------------------------------------- edge cases / errors
def test_oracle_edge_cases(orc):
    m, n = 10, 6
    c, r, v, b, lam = small_problem(m, n, [0, 0, 3, 0, 2, 10], seed=1)
    res = orc.run(m, c, r, v, b, lam, 6, 3, seed=0, x0=np.full(n, 0.5))
    # empty columns jump to 0 when lam > 0 (reading R#5)
    assert res.x[0] == 0.0 and res.x[1] == 0.0 and res.x[3] == 0.0
    res0 = orc.run(m, c, r, v, b, 0.0, 6, 3, seed=0, x0=np.full(n, 0.5))
    assert res0.x[0] == 0.5
    zero = orc.run(m, c, r, v, b, lam, 3, 0, seed=0)
    assert np.all(zero.x == 0) and np.allclose(zero.r, -b)
    with pytest.raises(ValueError):
        orc.run(m, c, r, v, b, lam, n + 1, 1, seed=0)
