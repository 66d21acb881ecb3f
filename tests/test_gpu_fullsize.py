"""Parity at BASELINE.json's full `huge` size (m = 1e8, n = 5e8, 5e9 nonzeros), in
the launch configuration bench.py times (AUTO -> the batched loop, tau = 2^18), and
for the packed loop.

The oracle cannot hold the whole run, but the first K iterations only ever touch
the columns S_0 .. S_{K-1} draw, and with x_0 = 0 every other column stays zero:
the oracle runs the same K iterations of alg:PCD1 on the
sub-matrix of those columns (b and r over all m rows) and must agree with the GPU
on x (touched columns), F and the whole maintained residual.  omega and the column
norms are checked against independent computations of their definitions."""
import numpy as np
import pytest
import torch

import oracle
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import F_RTOL, X_RTOL, to_host

pytestmark = pytest.mark.gpu

K = 24


def _subinstance(inst, tau, k_iters, seed):
    S = [oracle.sample(seed, k, tau, inst.n) for k in range(k_iters)]
    cols = np.unique(np.concatenate(S)).astype(np.int64)
    dev = inst.colptr.device
    ct = torch.from_numpy(cols).to(dev)
    starts = inst.colptr[ct]
    lens = inst.colptr[ct + 1] - starts
    total = int(lens.sum())
    offs = torch.cumsum(lens, 0) - lens
    idx = torch.repeat_interleave(starts - offs, lens) + torch.arange(total, device=dev)
    rows = inst.rowidx[idx].cpu().numpy()
    vals = inst.val[idx].cpu().numpy()
    colptr = np.zeros(inst.n + 1, dtype=np.int64)
    colptr[cols + 1] = lens.cpu().numpy()
    np.cumsum(colptr, out=colptr)
    return cols, colptr, rows, vals


def test_huge_full_size_first_iterations(gpu):
    cfg = I.CONFIGS["huge"]
    if torch.cuda.get_device_properties(gpu).total_memory < 150e9:
        pytest.skip("the huge config needs ~120 GB of device memory")
    inst = I.generate(cfg, seed=0, device=gpu)
    tau, seed = cfg.tau, 0
    prob = pcdm.Problem.from_instance(inst)
    # omega: the definition (max stored entries in a row) via torch.bincount,
    # in chunks of 2^28 entries (one bincount over all 5e9 entries returns wrong counts)
    counts = torch.zeros(inst.m, dtype=torch.int64, device=gpu)
    for p0 in range(0, inst.rowidx.numel(), 1 << 28):
        counts += torch.bincount(inst.rowidx[p0:p0 + (1 << 28)], minlength=inst.m)
    assert int(counts.sum()) == inst.rowidx.numel()
    assert prob.omega == int(counts.max())
    del counts
    # L_i = ||a_i||^2 on sampled columns, fp64 on the host
    L = torch.empty(inst.n, dtype=torch.float32, device=gpu)
    prob.col_norms(L)
    pick = torch.randint(0, inst.n, (4096,), device=gpu, generator=torch.Generator(device=gpu).manual_seed(1))
    Lh = to_host(L[pick])
    c = cfg.nnz_per_col
    vals = to_host(inst.val.view(inst.n, c)[pick]).astype(np.float64)
    np.testing.assert_allclose(Lh, (vals ** 2).sum(1).astype(np.float32), rtol=2e-7, atol=0)
    del L

    # AUTO (the batched loop: r is 400 MB, much larger than L2) and the packed loop
    runs = {}
    for variant, want in (("auto", "batched"), ("packed", "packed")):
        x = torch.zeros(inst.n, dtype=torch.float32, device=gpu)
        prob.run(x, tau, K, seed=seed, variant=variant)
        st = prob.stats()
        assert st["variant"] == pcdm.VARIANTS[want] and st["iters"] == K
        r_gpu = torch.empty(inst.m, dtype=torch.float32, device=gpu)
        prob.residual(r_gpu)
        runs[want] = (prob.objective(x), to_host(x), to_host(r_gpu))
        del x, r_gpu
    beta = prob.beta(tau)  # from the full matrix's omega (the sub-matrix's omega is smaller)
    assert abs(beta - oracle.beta(prob.omega, tau, inst.n)) <= 1e-15 * beta
    prob.close()

    cols, colptr, rows, vals = _subinstance(inst, tau, K, seed)
    b, lam, m = to_host(inst.b), inst.lam, inst.m
    del inst
    torch.cuda.empty_cache()
    res = oracle.run(m, colptr, rows, vals, b, lam, tau, K, seed, beta_override=beta)
    F_orc = oracle.objective(m, colptr, rows, vals, b, lam, res.x)
    untouched = np.ones(runs["packed"][1].size, dtype=bool)
    untouched[cols] = False
    xo = res.x[cols]
    scale = max(np.max(np.abs(xo)), 1e-30)
    for name, (F_gpu, xg, r_gpu) in runs.items():
        assert abs(F_gpu - F_orc) <= F_RTOL * abs(F_orc), (name, F_gpu, F_orc)
        # x: zero off the touched columns, oracle values on them
        assert not np.any(xg[untouched]), name
        assert np.max(np.abs(xg[cols].astype(np.float64) - xo)) <= X_RTOL * scale, name
        # the maintained residual over all 1e8 rows
        assert np.max(np.abs(r_gpu - res.r)) <= 1e-4 * np.max(np.abs(res.r)), name
