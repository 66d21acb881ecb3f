"""NEXT-2: Sec. 8.2 "theory versus reality".

The oracle reproduces the paper's observation that the tau-nice speedup factor of
tbl:upperbounds predicts the empirical iteration speedup on
matrices whose rows hold omega equal nonzeros; the CUDA path's iteration counts
to eps match the oracle's on the same instance (GPU test).
"""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import theory_vs_reality as T  # noqa: E402

from paper_1212_0873_b200 import instances as I

M, N, OM = 120, 40, 4
TAUS = (1, 2, 4, 8, 20, 40)


def test_equal_row_random_matrix_structure():
    c, r, v = I.equal_row_random_matrix(3000, 1000, 50, seed=3)
    c, r = c.numpy(), r.numpy()
    assert np.all(np.diff(c) == 150)                          # k = omega m / n ones per column
    assert np.all(np.bincount(r, minlength=3000) == 50)       # omega ones per row
    for i in range(0, 1000, 97):
        assert np.all(np.diff(r[c[i]:c[i + 1]]) > 0)
    assert np.all(v.numpy() == 1.0)


def _oracle_counts(orc, c, r, v, b, Fs):
    out = {}
    for tau in TAUS:
        def runner(x, k0, K, tau=tau):
            if K == 0:
                return x
            return orc.run(M, c, r, v, b, 0.0, tau, K, 0, x0=x.astype(np.float64), first_iter=k0,
                           ).x.astype(np.float32)
        obj = lambda x: orc.objective(M, c, r, v, b, 0.0, x.astype(np.float64))
        out[tau] = T.iters_to_eps(runner, obj, N, 1e-6, Fs)
    return out


def test_oracle_speedup_tracks_theory(orc):
    c, r, v, b, Fs = T.make_problem(M, N, OM, seed=0)
    assert Fs < 1e-9
    K = _oracle_counts(orc, c, r, v, b, Fs)
    for tau in TAUS[1:]:
        emp, th = K[1] / K[tau], T.theoretical_speedup(tau, OM, N)
        tol = 0.15 if tau <= 8 else 0.25
        assert abs(emp - th) <= tol * th, (tau, emp, th)
    # more processors never need more iterations here
    assert all(K[a] >= K[bb] for a, bb in zip(TAUS, TAUS[1:]))


@pytest.mark.gpu
def test_gpu_iteration_counts_match_oracle(gpu, orc):
    c, r, v, b, Fs = T.make_problem(M, N, OM, seed=0)
    K = _oracle_counts(orc, c, r, v, b, Fs)
    for tau in (1, 4, 40):
        prob, runner, objective = T.gpu_counter(c, r, v, b, M, tau)
        Kg = T.iters_to_eps(runner, objective, N, 1e-6, Fs)
        prob.close()
        assert abs(Kg - K[tau]) <= max(2, 0.03 * K[tau]), (tau, Kg, K[tau])
