"""NEXT-3: the L2-regularised logistic problem of Sec. 8.4 on the CUDA
path (pcdm_create_logistic) against the oracle (oracle.logistic_run), same
tolerances as the LASSO path: F within 1e-5 relative, ||dx||_inf <= 1e-4 ||x||_inf."""
import numpy as np
import pytest
import torch

import oracle
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import F_RTOL, X_RTOL, to_host

pytestmark = pytest.mark.gpu


def _labels(m, seed):
    return torch.from_numpy(np.where(np.random.default_rng(seed).normal(size=m) > 0, 1.0, -1.0).astype(np.float32))


def run_both_logistic(colptr, rowidx, val, y, lam, m, tau, iters, seed=0, variant="auto", sampling=None,
                      refresh_every=0, first_iter=0, x0=None):
    n = colptr.numel() - 1
    dev = torch.device("cuda:0")
    prob = pcdm.Problem(m, n, colptr.to(dev), rowidx.to(dev), val.to(dev), y.to(dev), lam, loss="logistic")
    x = torch.zeros(n, device=dev) if x0 is None else torch.as_tensor(x0, dtype=torch.float32).to(dev).clone()
    prob.run(x, tau, iters, seed=seed, variant=variant, refresh_every=refresh_every, first_iter=first_iter,
             sampling=None if sampling is None else pcdm.Sampling(*sampling))
    st = prob.stats()
    F = prob.objective(x)
    s_gpu = torch.empty(m, device=dev)
    prob.residual(s_gpu)
    L_gpu = torch.empty(n, device=dev)
    prob.col_norms(L_gpu)
    prob.close()
    c, r, v, yy = to_host(colptr), to_host(rowidx), to_host(val), to_host(y)
    res = oracle.logistic_run(m, c, r, v, yy, lam, tau, iters, seed, x0=None if x0 is None else np.asarray(x0, np.float64),
                              refresh_every=refresh_every, first_iter=first_iter,
                              sampling=None if sampling is None else oracle.Sampling(*sampling))
    Fo = oracle.logistic_objective(m, c, r, v, yy, lam, res.x)
    return dict(x=to_host(x).astype(np.float64), xo=res.x, F=F, Fo=Fo, st=st, s_gpu=to_host(s_gpu), res=res,
                L_gpu=to_host(L_gpu), c=c, r=r, v=v, y=yy)


def check(out):
    assert abs(out["F"] - out["Fo"]) <= F_RTOL * abs(out["Fo"]), (out["F"], out["Fo"])
    scale = max(np.max(np.abs(out["xo"])), 1e-30)
    assert np.max(np.abs(out["x"] - out["xo"])) <= X_RTOL * scale


@pytest.mark.parametrize("variant", ["auto", "packed", "grid", "block"])
def test_logistic_small_config(gpu, variant):
    colptr, rowidx, val, y, lam = I.generate_logistic("logistic_small", seed=0)
    out = run_both_logistic(colptr, rowidx, val, y, lam, 20_000, 1024, 300, variant=variant)
    check(out)
    # the library's L and margins
    np.testing.assert_allclose(out["L_gpu"], oracle.logistic_L(out["c"], out["v"]).astype(np.float32), rtol=2e-7)
    s_x = oracle.margins(20_000, out["c"], out["r"], out["v"], out["y"], out["x"])
    assert np.max(np.abs(out["s_gpu"] - s_x)) <= 1e-4 * max(1.0, np.max(np.abs(s_x)))


@pytest.mark.parametrize("variant", ["smem", "grid"])
def test_logistic_ragged_samplings_and_edges(gpu, variant):
    m, n = 600, 400
    lens = np.random.default_rng(5).integers(0, 20, size=n)
    lens[:3] = 0
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=6)
    y = _labels(m, 7)
    x0 = np.random.default_rng(8).normal(size=n) * (np.arange(n) % 4 == 0)
    for tau, lam, smp in ((1, 0.5, None), (37, 1.0, None), (400, 0.1, None), (37, 0.0, None),
                          (64, 1.0, ("binomial", 64, 0.5, None)), (50, 1.0, ("independent", 50, 1.0, None))):
        out = run_both_logistic(colptr, rowidx, val, y, lam, m, tau, 80, seed=tau, variant=variant, sampling=smp,
                                x0=x0, first_iter=3)
        check(out)


def test_logistic_errors(gpu):
    colptr, rowidx, val = I.random_csc(50, 40, np.full(40, 3), seed=1)
    y = _labels(50, 2)
    y[7] = 0.5
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.Problem(50, 40, colptr.to(gpu), rowidx.to(gpu), val.to(gpu), y.to(gpu), 1.0, loss="logistic")
    assert e.value.status == pcdm.PCDM_EINVAL and "labels" in e.value.message
    y[7] = 1.0
    prob = pcdm.Problem(50, 40, colptr.to(gpu), rowidx.to(gpu), val.to(gpu), y.to(gpu), 1.0, loss="logistic")
    with pytest.raises(pcdm.PCDMError) as e:
        prob.run_async(torch.zeros(40, device=gpu), 100)
    assert e.value.status == pcdm.PCDM_EINVAL
    # objective at 0: m log 2 (Sec. 8.4 F(x0) = d log 2 for x0 = 0)
    assert prob.objective(torch.zeros(40, device=gpu)) == pytest.approx(50 * np.log(2.0), rel=1e-12)
    prob.close()
