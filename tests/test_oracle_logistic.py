"""Pins for the oracle's L2-regularised logistic regression (
Sec. 8.4, logistic loss of tbl:ML3 PAPER.md:68, reading R21).

Checked against: finite differences of F (gradient), the quadratic upper bound
with L_i = 1/4||a_i||^2 and its tightness at zero margins, brute-force
minimisation of the block model, monotone serial steps, the expected-decrease
inequality eq:1 by exact enumeration, and the optimum of the (strongly convex)
problem found by scipy's L-BFGS.
"""
import itertools

import numpy as np
import pytest
from scipy import optimize

from paper_1212_0873_b200 import instances as I


def small(m=25, n=12, lens=None, seed=0, lam=0.3):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 7, size=n) if lens is None else lens
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=seed)
    c, r, v = colptr.numpy(), rowidx.numpy(), val.numpy()
    y = np.where(rng.normal(size=m) > 0, 1.0, -1.0).astype(np.float32)
    A = np.zeros((m, n))
    for i in range(n):
        A[r[c[i]:c[i + 1]], i] = v[c[i]:c[i + 1]]
    return c, r, v, y, lam, A


def F_dense(A, y, lam, x):
    s = y * (A @ x)
    return float(np.sum(np.logaddexp(0.0, -s)) + lam * x @ x)


def test_objective_and_gradient(orc):
    c, r, v, y, lam, A = small(seed=1)
    m, n = A.shape
    rng = np.random.default_rng(2)
    for _ in range(5):
        x = rng.normal(size=n)
        assert orc.logistic_objective(m, c, r, v, y, lam, x) == pytest.approx(F_dense(A, y, lam, x), rel=1e-13)
        s = orc.margins(m, c, r, v, y, x)
        for i in range(n):
            h = 1e-6
            e = np.zeros(n)
            e[i] = h
            fd = (F_dense(A, y, 0.0, x + e) - F_dense(A, y, 0.0, x - e)) / (2 * h)
            assert orc.logistic_grad_i(c, r, v, y, s, i) == pytest.approx(fd, rel=1e-6, abs=1e-8)


def test_block_lipschitz_bound_and_tightness(orc):
    c, r, v, y, lam, A = small(seed=3)
    m, n = A.shape
    L = orc.logistic_L(c, v)
    assert np.allclose(L, 0.25 * (A ** 2).sum(0))
    rng = np.random.default_rng(4)
    f = lambda z: F_dense(A, y, 0.0, z)
    for _ in range(20):
        x = rng.normal(size=n) * 2
        s = orc.margins(m, c, r, v, y, x)
        i = int(rng.integers(n))
        g = orc.logistic_grad_i(c, r, v, y, s, i)
        for t in (-3.0, -0.5, 0.1, 2.0):
            e = np.zeros(n)
            e[i] = t
            assert f(x + e) <= f(x) + g * t + 0.5 * L[i] * t * t + 1e-12
    # at zero margins the curvature along e_i is exactly L_i (only the rows of column i vary)
    for i in range(n):
        a, yy = A[:, i], y.astype(np.float64)
        fi = lambda t: float(np.sum(np.logaddexp(0.0, -yy * a * t)))
        t = 1e-3
        curv = (fi(t) + fi(-t) - 2 * fi(0.0)) / t ** 2
        assert curv == pytest.approx(L[i], rel=1e-4)


def test_step_is_exact_model_minimiser(orc):
    rng = np.random.default_rng(5)
    for _ in range(200):
        x, g, s, lam = rng.normal(), rng.normal() * 3, rng.uniform(0.1, 5), rng.uniform(0, 2)
        xp = orc.logistic_step(x, g, s, lam)
        model = lambda t: g * t + 0.5 * s * t * t + lam * (x + t) ** 2
        best = optimize.minimize_scalar(model, tol=1e-12).x
        assert xp - x == pytest.approx(best, rel=1e-7, abs=1e-7)
        t = xp - x                                    # stationarity of the strictly convex model
        assert abs(g + s * t + 2 * lam * (x + t)) <= 1e-12 * (abs(g) + s * abs(t) + 2 * lam * abs(x + t) + 1)
    assert orc.logistic_step(0.7, 1.0, 0.0, 0.0) == 0.7      # empty column, lambda = 0


def test_serial_steps_monotone_and_converge_to_lbfgs(orc):
    c, r, v, y, lam, A = small(m=40, n=15, seed=6)
    m, n = A.shape
    x = np.zeros(n)
    F = orc.logistic_objective(m, c, r, v, y, lam, x)
    for k in range(300):
        x = orc.logistic_run(m, c, r, v, y, lam, 1, 1, seed=9, x0=x, first_iter=k).x
        Fn = orc.logistic_objective(m, c, r, v, y, lam, x)
        assert Fn <= F + 1e-12
        F = Fn
    ref = optimize.minimize(lambda z: F_dense(A, y, lam, z), np.zeros(n),
                            jac=lambda z: -A.T @ (y / (1 + np.exp(y * (A @ z)))) + 2 * lam * z,
                            method="L-BFGS-B", options={"gtol": 1e-12, "ftol": 1e-15, "maxiter": 10000}).x
    for tau in (1, 4, 15):
        res = orc.logistic_run(m, c, r, v, y, lam, tau, 30000 // tau, seed=2)
        assert np.max(np.abs(res.x - ref)) <= 1e-6


def test_expected_decrease_eq1_exact_enumeration(orc):
    # eq:1 with Omega = lambda ||.||^2:
    # E F(x + h_[S]) <= (1 - tau/n) F(x) + (tau/n) H_{beta,L}(x, h), h = h(x) for all blocks
    c, r, v, y, lam, A = small(m=14, n=8, lens=[3, 4, 2, 5, 3, 1, 4, 2], seed=11)
    m, n = A.shape
    om = orc.omega(m, r)
    L = orc.logistic_L(c, v)
    rng = np.random.default_rng(3)
    for tau in (2, 3, 8):
        beta = orc.beta(om, tau, n)
        x = rng.normal(size=n)
        h = orc.logistic_run(m, c, r, v, y, lam, n, 1, seed=0, x0=x, beta_override=beta).x - x
        s = orc.margins(m, c, r, v, y, x)
        grad = np.array([orc.logistic_grad_i(c, r, v, y, s, i) for i in range(n)])
        Fx = F_dense(A, y, lam, x)
        H = F_dense(A, y, 0.0, x) + grad @ h + 0.5 * beta * np.sum(L * h * h) + lam * np.sum((x + h) ** 2)
        vals = []
        for S in itertools.combinations(range(n), tau):
            z = x.copy()
            z[list(S)] += h[list(S)]
            vals.append(F_dense(A, y, lam, z))
        a = tau / n
        assert np.mean(vals) <= (1 - a) * Fx + a * H + 1e-12
        assert (1 - a) * Fx + a * H <= Fx + 1e-12


def test_logistic_instance_shape():
    colptr, rowidx, val, y, lam = I.generate_logistic("logistic_small", seed=0)
    assert colptr[-1] == rowidx.numel() == 30_000 * 19
    assert set(np.unique(y.numpy()).tolist()) == {-1.0, 1.0}
    assert lam == 1.0
