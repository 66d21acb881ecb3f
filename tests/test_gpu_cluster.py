"""CLUSTER variant (kernels_cluster.cu): the synchronous PCDM1 iteration
(alg:PCD1 PAPER.md:177-186) with r split over one thread-block cluster's shared
memories and two hardware cluster barriers per iteration.  Same arithmetic as the
packed loop, so the north_star tolerances against the oracle apply: F within 1e-5
relative, ||dx||_inf <= 1e-4 ||x||_inf, maintained residual equal to the oracle's."""
import numpy as np
import pytest
import torch

from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import assert_parity, run_both
from test_gpu_logistic import _labels, check, run_both_logistic

pytestmark = pytest.mark.gpu


def _ragged(m, n, lens, seed, lam_frac=0.1):
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=seed)
    b = I.random_b(m, seed=seed)
    return colptr, rowidx, val, b, I.lam_for(colptr, rowidx, val, b, lam_frac)


def _check_r(out):
    np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0, atol=1e-4 * np.max(np.abs(out["res"].r)))


def test_cluster_medium_config_full_run(gpu, monkeypatch):
    # BASELINE configs[1]: medium, tau = 1024, 1e4 iterations; AUTO picks the cluster loop
    # when PCDM_CLUSTER=1
    monkeypatch.setenv("PCDM_CLUSTER", "1")
    inst = I.generate("medium", seed=0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 1024, 10_000, seed=0)
    assert out["stats"]["variant"] == pcdm.VARIANTS["cluster"]
    assert out["stats"]["grid_ctas"] in (2, 4, 8, 16)
    assert_parity(out)
    _check_r(out)


@pytest.mark.parametrize("lens_kind", ["uniform10", "uniform20", "ragged"])
def test_cluster_matches_oracle(gpu, lens_kind):
    m, n = 5000, 4000
    rng = np.random.default_rng(3)
    lens = {"uniform10": np.full(n, 10), "uniform20": np.full(n, 20),
            "ragged": rng.integers(0, 62, size=n)}[lens_kind]
    if lens_kind == "ragged":
        lens[:5] = 0
        lens[5] = 62
    c, r, v, b, lam = _ragged(m, n, lens, 8, lam_frac=0.05)
    x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 7 == 0)
    # tau up to n: several slots per group and per-CTA step lists of several entries
    for tau, iters, refresh in ((1, 300, 0), (64, 200, 0), (1000, 40, 7), (4000, 5, -1)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="cluster", x0=x0, refresh_every=refresh)
        assert out["stats"]["variant"] == pcdm.VARIANTS["cluster"]
        assert_parity(out)
        _check_r(out)


@pytest.mark.parametrize("x_in_block", ["1", "0"])
def test_cluster_x_storage_chunks_and_hot_rows(gpu, monkeypatch, x_in_block):
    monkeypatch.setenv("PCDM_X_IN_BLOCK", x_in_block)
    monkeypatch.setenv("PCDM_CHUNK", "7")
    monkeypatch.setenv("PCDM_ITER_CHUNK", "7")
    inst = I.generate(I.InstanceConfig("zipf_small", 20_000, 20_000, 20, 200, rows="zipf"), seed=0)
    for tau, iters in ((2048, 60), (200, 200)):
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=tau,
                       variant="cluster")
        assert out["stats"]["iter_launches"] >= iters // 7
        assert_parity(out)
        _check_r(out)


SAMPLINGS = [("independent", 700, 1.0, None), ("binomial", 500, 0.6, None),
             ("du", 40, 1.0, list(np.random.default_rng(9).dirichlet(np.ones(41))))]


@pytest.mark.parametrize("spec", SAMPLINGS, ids=lambda s: "%s-%d" % (s[0], s[1]))
def test_cluster_samplings(gpu, spec):
    c, r, v, b, lam = _ragged(3000, 2000, np.random.default_rng(1).integers(1, 25, size=2000), 3)
    out = run_both(c, r, v, b, lam, 3000, spec[1], 120, seed=4, variant="cluster", sampling=spec)
    assert_parity(out)


def test_cluster_logistic(gpu):
    colptr, rowidx, val, y, lam = I.generate_logistic("logistic_small", seed=0)
    out = run_both_logistic(colptr, rowidx, val, y, lam, 20_000, 1024, 300, variant="cluster")
    check(out)
    m, n = 600, 400
    lens = np.random.default_rng(5).integers(0, 20, size=n)
    lens[:3] = 0
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=6)
    y = _labels(m, 7)
    x0 = np.random.default_rng(8).normal(size=n) * (np.arange(n) % 4 == 0)
    for tau, lam in ((37, 1.0), (400, 0.1)):
        check(run_both_logistic(colptr, rowidx, val, y, lam, m, tau, 80, seed=tau, variant="cluster", x0=x0,
                                first_iter=3))


def test_cluster_rejected_when_r_does_not_fit(gpu):
    m, n = 4_000_000, 2000
    inst = I.generate(I.InstanceConfig("tall", m, n, 4, 20), seed=0)
    prob = pcdm.Problem.from_instance(inst.to(gpu))
    x = torch.zeros(n, device=gpu)
    with pytest.raises(pcdm.PCDMError) as e:
        prob.run(x, 16, 1, variant="cluster")
    assert e.value.status == pcdm.PCDM_EINVAL
    prob.run(x, 16, 1)  # AUTO falls back to the grid loop
    assert prob.stats()["variant"] == pcdm.VARIANTS["packed"]
    prob.close()
