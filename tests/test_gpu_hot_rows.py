"""Hot rows of the packed loop (kernels_packed.cu): on skewed (Zipf) row
distributions the rows stored in many columns are encoded in the blocks and
gathered from a per-CTA shared-memory copy of r_k.  The arithmetic is unchanged
(same synchronous PCDM1 step, alg:PCD1 PAPER.md:177-186), so the oracle tolerances
of the north_star apply: F within 1e-5 relative, ||dx||_inf <= 1e-4 ||x||_inf."""
import numpy as np
import pytest
import torch

import oracle
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import assert_parity, run_both, to_host
from test_gpu_logistic import _labels, check, run_both_logistic

pytestmark = pytest.mark.gpu

ZIPF_SMALL = I.InstanceConfig("zipf_small", 20_000, 20_000, 20, 200, rows="zipf")


@pytest.fixture(scope="module")
def zipf():
    return I.generate(ZIPF_SMALL, seed=0)


def _hot_count(inst, gpu, tau=None):
    prob = pcdm.Problem.from_instance(inst.to(gpu))
    x = torch.zeros(inst.n, device=gpu)
    prob.run(x, tau or inst.n, 1, variant="packed")
    h = prob.stats()["hot_rows"]
    prob.close()
    return h


def test_hot_row_selection(gpu, zipf, monkeypatch):
    # rows stored >= max(64, 32 x mean) times; mean 20 -> threshold 640
    counts = oracle.row_counts(zipf.m, to_host(zipf.rowidx))
    want = int(np.sum(counts >= 640))
    assert 0 < want <= 2048
    assert _hot_count(zipf, gpu) == want
    monkeypatch.setenv("PCDM_HOT_MAX", "5")
    assert _hot_count(zipf, gpu) == 5
    monkeypatch.setenv("PCDM_HOT_ROWS", "0")
    assert _hot_count(zipf, gpu) == 0
    # uniform rows: none
    monkeypatch.delenv("PCDM_HOT_ROWS")
    monkeypatch.delenv("PCDM_HOT_MAX")
    assert _hot_count(I.generate("tiny", seed=0), gpu) == 0
    # the run caches them only when the hottest row is read >= 1024 times per iteration
    top = int(counts.max())
    assert _hot_count(zipf, gpu, tau=(1024 * zipf.n) // top - 1) == 0
    assert _hot_count(zipf, gpu, tau=(1024 * zipf.n + top - 1) // top) == want


@pytest.mark.parametrize("stage", ["0", "1"], ids=["scatter-global", "scatter-staged"])
@pytest.mark.parametrize("one_barrier", ["1", "0"])
@pytest.mark.parametrize("hot_max,cache", [(None, "1"), ("5", "1"), (None, "0")])
def test_hot_rows_parity(gpu, zipf, monkeypatch, one_barrier, hot_max, cache, stage):
    # stage: hot-row scatters accumulated per CTA in shared memory (one-barrier scheme)
    monkeypatch.setenv("PCDM_ONE_BARRIER", one_barrier)
    monkeypatch.setenv("PCDM_HOT_CACHE", cache)
    monkeypatch.setenv("PCDM_HOT_STAGE", stage)
    if hot_max:
        monkeypatch.setenv("PCDM_HOT_MAX", hot_max)
    inst = zipf
    for tau, iters in ((64, 400), (2048, 120), (inst.n, 6)):
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=tau,
                       variant="packed")
        assert (out["stats"]["hot_rows"] > 0) == (cache == "1")
        assert_parity(out)
    # a nonzero start: every iteration scatters into the hot rows
    x0 = np.random.default_rng(1).normal(size=inst.n) * (np.arange(inst.n) % 3 == 0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 1000, 60, seed=3,
                   variant="packed", x0=x0, refresh_every=25)
    assert_parity(out)


@pytest.mark.parametrize("stage", ["0", "1"], ids=["scatter-global", "scatter-staged"])
def test_hot_rows_logistic(gpu, zipf, monkeypatch, stage):
    # logistic: every visited coordinate steps, so every iteration scatters into the hot rows
    monkeypatch.setenv("PCDM_HOT_STAGE", stage)
    y = _labels(zipf.m, 3)
    out = run_both_logistic(zipf.colptr, zipf.rowidx, zipf.val, y, 1.0, zipf.m, 2048, 100, variant="packed")
    assert out["st"]["hot_rows"] > 0
    check(out)


def test_hot_rows_async_invariant(gpu, zipf):
    # the asynchronous loop decodes hot entries through the global table: r == Ax - b
    inst = zipf
    prob = pcdm.Problem.from_instance(inst.to(gpu))
    x = torch.zeros(inst.n, device=gpu)
    prob.run_async(x, 20 * inst.n, seed=2)
    assert prob.stats()["nonzero_deltas"] > 0
    rg = torch.empty(inst.m, device=gpu)
    prob.residual(rg)
    c, r, v, b = inst.numpy()
    rx = oracle.residual(inst.m, c, r, v, b, to_host(x).astype(np.float64))
    assert np.max(np.abs(to_host(rg) - rx)) <= 1e-4 * max(1.0, np.max(np.abs(rx)))
    prob.close()
