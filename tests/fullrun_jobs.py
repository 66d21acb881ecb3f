"""Full-length oracle runs for the parity tests of tests/test_gpu_fullrun.py
(test infrastructure).

The oracle is serial (plain C, fp64) and the benchmarked run lengths take it
minutes (large: 2000 iterations of tau = 65536; skewed: 10^4 iterations per tau;
huge: 500 iterations of tau = 2^18).  So when the full-run tests are selected,
the `gpu` session fixture calls start() once: the instances are generated on
the GPU (an instance is a function of (config, seed, device type), so both
sides must use the GPU-built arrays), copied to the host, and each oracle run is
forked into its own process, which works on the host arrays only (numpy + the
oracle's ctypes library; it never touches CUDA) and leaves its result in an
.npz.  The rest of the GPU suite runs meanwhile; the full-run tests then wait
for their job.

Nothing here comes from the CUDA path: the columns the huge run touches come
from the oracle's own sampler, omega from the oracle's own count over the full
matrix, and every expected value from oracle.run / oracle.objective.
"""
from __future__ import annotations

import os
import shutil
import tempfile

import numpy as np

from oracle.background import Job as _Job

HUGE_ITERS = 500
LARGE_ITERS = 2000
SKEWED_ITERS = 10_000
SKEWED_TAUS = (1 << 8, 1 << 12, 1 << 16)

_jobs = {}
_tmp = None


def Job(name, fn):
    return _Job(name, fn, _tmp)


def get(name):
    if name not in _jobs:
        raise KeyError("oracle job %s was not started (run the module under the `gpu` fixture)" % name)
    return _jobs[name]


def started():
    return bool(_jobs)


def _oracle_run_job(m, colptr, rowidx, val, b, lam, tau, iters, omega_override=None, keep_x_at=None):
    import oracle

    def fn():
        res = oracle.run(m, colptr, rowidx, val, b, lam, tau, iters, 0, omega_override=omega_override)
        F = oracle.objective(m, colptr, rowidx, val, b, lam, res.x)
        x = res.x if keep_x_at is None else res.x[keep_x_at]
        return dict(x=x, r=res.r, F=np.float64(F), omega=np.int64(res.omega), beta=np.float64(res.beta),
                    loop_seconds=np.float64(res.loop_seconds))
    return fn


def start(device):
    """Generate the full-run instances on `device` and fork their oracle runs."""
    global _tmp
    if _jobs:
        return
    import torch

    import oracle
    from paper_1212_0873_b200 import instances as I

    oracle.build()
    _tmp = tempfile.mkdtemp(prefix="pcdm_fullrun_")

    # skewed: one instance (seed 0) for every tau
    inst = I.generate("skewed", seed=0, device=device)
    c, r, v, b = inst.numpy()
    for tau in SKEWED_TAUS:
        _jobs["skewed_%d" % tau] = Job("skewed_%d" % tau,
                                       _oracle_run_job(inst.m, c, r, v, b, inst.lam, tau, SKEWED_ITERS))
    del inst, c, r, v, b

    cfg = I.CONFIGS["large"]
    inst = I.generate(cfg, seed=0, device=device)
    c, r, v, b = inst.numpy()
    _jobs["large"] = Job("large", _oracle_run_job(inst.m, c, r, v, b, inst.lam, cfg.tau, LARGE_ITERS))
    del inst, c, r, v, b
    torch.cuda.empty_cache()

    # huge: only the columns S_0..S_499 touch can become nonzero (x_0 = 0); the
    # oracle runs the same iterations on that sub-matrix, with omega (hence beta)
    # counted by the oracle over all 5e9 entries of the full matrix.
    cfg = I.CONFIGS["huge"]
    if torch.cuda.get_device_properties(device).total_memory >= 150e9:
        inst = I.generate(cfg, seed=0, device=device)
        S = oracle.samples(0, 0, HUGE_ITERS, cfg.tau, cfg.n)
        cols = np.unique(S)
        np.save(os.path.join(_tmp, "huge_slots.npy"), S[[0, 1, HUGE_ITERS // 2, HUGE_ITERS - 1]])
        del S
        colptr, rows, vals = I.column_subset(inst.colptr, inst.rowidx, inst.val, cols)
        b = inst.b.cpu().numpy()
        full_rows = inst.rowidx.cpu().numpy()
        m, lam = inst.m, inst.lam
        del inst
        torch.cuda.empty_cache()
        def huge_fn():
            om = oracle.omega(m, full_rows)  # O1 over the full matrix
            out = _oracle_run_job(m, colptr, rows, vals, b, lam, cfg.tau, HUGE_ITERS, omega_override=om,
                                  keep_x_at=cols)()
            out["omega_full"] = np.int64(om)
            out["cols"] = cols
            return out
        _jobs["huge"] = Job("huge", huge_fn)
        del full_rows, colptr, rows, vals, b


def slots_path(name):
    return os.path.join(_tmp, name + "_slots.npy")


def cleanup():
    for j in _jobs.values():
        j.kill()
    if _tmp:
        shutil.rmtree(_tmp, ignore_errors=True)
