#!/usr/bin/env python
"""Theory versus reality (Sec. 8.2).

Minimise f(x) = 1/2||Ax - b||^2 (lambda = 0) with A in R^{3000 x 1000} whose every
row holds exactly omega equal nonzeros (instances.equal_row_random_matrix, built on the
DSO tightness construction of PAPER.md:697-703), count the PCDM1 iterations
needed to get within eps = 1e-6 of the optimal value with the tau-nice sampling,
and compare the empirical speedup

    iters(serial, tau = 1) / iters(tau-nice)

with the theoretical parallelization speedup factor of tbl:upperbounds
(PAPER.md:1103): s = tau / (1 + (omega - 1)(tau - 1) / max(1, n - 1)).

b = A x* with x* ~ N(0,1) (consistent system, F* = 0 up to the fp32 rounding of
b; F* is computed by a dense fp64 least-squares solve).  The paper does not
print its b; this is reading R19.

    python tools/theory_vs_reality.py [--omegas 5 10 50 100] [--taus ...] [--out FILE]

Runs the CUDA path through the public API (paper_1212_0873_b200.pcdm); the
iteration count to eps is found exactly by doubling + bisection with resumed
runs (first_iter keeps the same sample stream).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1212_0873_b200 import instances as I  # noqa: E402


def make_problem(m=3000, n=1000, omega=5, seed=0):
    """(colptr, rowidx, val, b fp32, F*) for the Sec. 8.2 instance."""
    colptr, rowidx, val = I.equal_row_random_matrix(m, n, omega, seed=seed)
    c, r, v = colptr.numpy(), rowidx.numpy(), val.numpy()
    A = np.zeros((m, n))
    for i in range(n):
        A[r[c[i]:c[i + 1]], i] = v[c[i]:c[i + 1]]
    xs = np.random.default_rng(seed + 1).normal(size=n)
    b = (A @ xs).astype(np.float32)
    sol, *_ = np.linalg.lstsq(A, b.astype(np.float64), rcond=None)
    Fstar = 0.5 * float(np.sum((A @ sol - b.astype(np.float64)) ** 2))
    return c, r, v, b, Fstar


def theoretical_speedup(tau, omega, n):
    """tbl:upperbounds, tau-nice row."""
    return tau / (1.0 + (omega - 1) * (tau - 1) / max(1, n - 1))


def iters_to_eps(runner, objective, n, eps, Fstar, max_iters=1 << 24):
    """Smallest K with F(x_K) - F* <= eps.  runner(x, k0, K) runs iterations
    k0..k0+K-1 in place on x (float array), objective(x) -> F.  Doubling finds a
    bracket, bisection (re-running from the saved iterate) the exact K.  Returns
    None if F stops moving above eps (the fp32 iterate's floor: x_i + delta_i
    rounds back to x_i) or max_iters is reached."""
    x = np.zeros(n, dtype=np.float32)
    F = objective(x)
    if F - Fstar <= eps:
        return 0
    done, step = 0, 1
    while True:
        if done >= max_iters:
            return None
        saved = x.copy()
        x = runner(x, done, step)
        Fnew = objective(x)
        if step >= 1024 and Fnew >= F:
            return None
        F = Fnew
        if F - Fstar <= eps:
            lo, hi = 0, step          # crossing in (done + lo, done + hi]
            while hi - lo > 1:
                mid = (lo + hi) // 2
                y = runner(saved.copy(), done, mid)
                if objective(y) - Fstar <= eps:
                    hi = mid
                else:
                    lo = mid
            return done + hi
        done += step
        step *= 2


def gpu_counter(c, r, v, b, m, tau, seed=0):
    import torch
    from paper_1212_0873_b200 import pcdm
    dev = torch.device("cuda:0")
    n = len(c) - 1
    prob = pcdm.Problem(m, n, torch.from_numpy(c).to(dev), torch.from_numpy(r).to(dev),
                        torch.from_numpy(v).to(dev), torch.from_numpy(b).to(dev), 0.0)

    def runner(x, k0, K):
        xd = torch.from_numpy(x).to(dev)
        if K > 0:
            prob.run(xd, tau, K, seed=seed, first_iter=k0)  # default refresh R = ceil(2n/tau)
        return xd.cpu().numpy()

    def objective(x):
        return prob.objective(torch.from_numpy(x).to(dev))

    return prob, runner, objective


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--omegas", type=int, nargs="*", default=[5, 10, 50, 100])
    ap.add_argument("--taus", type=int, nargs="*", default=[1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1000])
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from paper_1212_0873_b200 import build, pcdm
    build.build()
    pcdm.load()
    m, n = 3000, 1000
    rows = []
    for om in args.omegas:
        c, r, v, b, Fstar = make_problem(m, n, om)
        serial = None
        for tau in args.taus:
            prob, runner, objective = gpu_counter(c, r, v, b, m, tau)
            K = iters_to_eps(runner, objective, n, args.eps, Fstar)
            prob.close()
            if tau == 1:
                serial = K
            row = {"omega": om, "tau": tau, "iters": K, "F_star": Fstar, "eps": args.eps,
                   "empirical_speedup": (serial / K) if (serial and K) else None,
                   "theoretical_speedup": theoretical_speedup(tau, om, n)}
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for row in rows:
                f.write(json.dumps(row) + "\n")


if __name__ == "__main__":
    main()
