"""The RAGGED packed layout (kernels_ragged.cu): a warp, sub-warp (2..32 lanes) or a
whole CTA per sampled column, by its number of nonzeros, with the slot arrays
binned by class after the sampler.  Same synchronous PCDM1 iteration (alg:PCD1,
PAPER.md:177-186) as every other loop: checked against the oracle at the
north_star tolerances on power-law column lengths (Pareto tail, longest column
12 000 entries: the KDDB-like shape of PAPER.md:1388-1392), on forced-ragged
layouts of other matrices, with refreshes, resumes, host x, hot rows, every
doubly uniform sampling and the logistic loss."""
import numpy as np
import pytest
import torch

import oracle
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import assert_parity, run_both, to_host

pytestmark = pytest.mark.gpu


def _ragged(m, n, lens, seed, lam_frac=0.1):
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=seed)
    b = I.random_b(m, seed=seed)
    return colptr, rowidx, val, b, I.lam_for(colptr, rowidx, val, b, lam_frac)


def _check_r(out):
    np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0, atol=1e-4 * np.max(np.abs(out["res"].r)))


@pytest.fixture(scope="module")
def zipf_cols():
    inst = I.generate("ragged_small", seed=0)
    lens = np.diff(inst.colptr.numpy())
    # every class: 2, 4, 8, 16, 32 lanes and CTA-long columns
    assert lens.max() >= 10_000 and all(c > 100 for c in np.histogram(lens, [0, 3, 7, 15, 31, 63, 1e9])[0])
    return inst


@pytest.mark.parametrize("bulk", ["0", "1"], ids=["ld-global", "bulk-staged"])
@pytest.mark.parametrize("variant", ["auto", "packed"])
def test_ragged_power_law_columns(gpu, zipf_cols, monkeypatch, variant, bulk):
    # bulk: CTA-long column slices staged in shared memory by cp.async.bulk (pieces of 4096
    # entries; the 12000-entry column takes three)
    monkeypatch.setenv("PCDM_BULK_STAGE", bulk)
    inst = zipf_cols
    x0 = np.random.default_rng(2).normal(size=inst.n) * (np.arange(inst.n) % 9 == 0)
    for tau, iters, refresh in ((1, 400, 0), (16, 300, 0), (256, 400, 0), (2000, 30, 5), (inst.n, 6, -1)):
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=tau,
                       variant=variant, x0=x0 if tau != 256 else None, refresh_every=refresh)
        st = out["stats"]
        assert st["variant"] == pcdm.VARIANTS["packed"] and st["lanes_per_column"] == 0, st
        assert_parity(out)
        _check_r(out)


def test_ragged_config_from_zero(gpu, zipf_cols):
    inst = zipf_cols
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, inst.cfg.tau, inst.cfg.iters, seed=0)
    assert out["stats"]["lanes_per_column"] == 0
    assert_parity(out)
    assert out["stats"]["nonzero_deltas"] > 0


@pytest.mark.parametrize("bulk", ["0", "1"], ids=["ld-global", "bulk-staged"])
@pytest.mark.parametrize("lens_kind", ["uniform10", "mixed", "one_long"])
def test_forced_ragged_layout(gpu, monkeypatch, lens_kind, bulk):
    # PCDM_LAYOUT=ragged (read at create) on matrices the uniform layout would take
    monkeypatch.setenv("PCDM_LAYOUT", "ragged")
    monkeypatch.setenv("PCDM_BULK_STAGE", bulk)
    m, n = 9000, 3000
    rng = np.random.default_rng(5)
    lens = {"uniform10": np.full(n, 10), "mixed": rng.integers(0, 70, size=n),
            "one_long": np.full(n, 3)}[lens_kind]
    lens[:4] = 0
    if lens_kind == "one_long":
        lens[16] = 4096 * 2 + 1  # CTA-long: three bulk pieces, the last one entry
        lens[17] = 4999
        lens[18] = 63
        lens[19] = 62
    c, r, v, b, lam = _ragged(m, n, lens, 8, lam_frac=0.05)
    x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 7 == 0)
    for tau, iters, refresh in ((1, 300, 0), (64, 200, 0), (1000, 40, 7), (n, 5, -1)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="packed", x0=x0, refresh_every=refresh)
        assert out["stats"]["lanes_per_column"] == 0
        assert_parity(out)
        _check_r(out)


def test_ragged_rejects_uniform_only_loops(gpu, zipf_cols):
    inst = zipf_cols
    prob = pcdm.Problem.from_instance(inst.to(gpu))
    x = torch.zeros(inst.n, device=gpu)
    for variant in ("batched",):
        with pytest.raises(pcdm.PCDMError) as e:
            prob.run(x, 8, 1, variant=variant)
        assert e.value.status == pcdm.PCDM_EINVAL
    with pytest.raises(pcdm.PCDMError) as e:
        prob.run_async(x, 100)
    assert e.value.status == pcdm.PCDM_EINVAL
    prob.close()


@pytest.mark.parametrize("kind", ["independent", "binomial", "du"])
def test_ragged_other_samplings(gpu, zipf_cols, kind):
    inst = zipf_cols
    tau = 128
    q = None
    if kind == "du":
        q = np.zeros(tau + 1)
        q[[1, 40, 128]] = [0.2, 0.5, 0.3]
    spec = (kind, tau, 0.5 if kind == "binomial" else 1.0, q)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, 200, seed=3,
                   variant="packed", sampling=spec)
    assert abs(out["beta_gpu"] - out["res"].beta) <= 1e-12 * out["res"].beta
    assert_parity(out)


def test_ragged_resume_and_host_x(gpu, zipf_cols):
    inst = zipf_cols
    c, r, v, b = inst.numpy()
    tau, k1, k2 = 64, 150, 170
    res = oracle.run(inst.m, c, r, v, b, inst.lam, tau, k1 + k2, 7)
    F_orc = oracle.objective(inst.m, c, r, v, b, inst.lam, res.x)
    with pcdm.Problem.from_instance(inst.to(gpu)) as prob:
        # device x in two runs (resume continues the sample stream) ...
        x = torch.zeros(inst.n, device=gpu)
        prob.run(x, tau, k1, seed=7)
        prob.run(x, tau, k2, seed=7, first_iter=k1)
        assert abs(prob.objective(x) - F_orc) <= 1e-5 * abs(F_orc)
        xg = to_host(x).astype(np.float64)
        assert np.max(np.abs(xg - res.x)) <= 1e-4 * np.max(np.abs(res.x))
        # ... and a pinned host x through the compact copy-back
        xh = torch.zeros(inst.n).pin_memory()
        prob.run(xh, tau, k1 + k2, seed=7)
        assert prob.stats()["lanes_per_column"] == 0
        assert np.max(np.abs(xh.numpy().astype(np.float64) - res.x)) <= 1e-4 * np.max(np.abs(res.x))


def test_ragged_hot_rows(gpu, monkeypatch):
    # Zipf rows on ragged columns: hot-row encoding in the ragged blocks, with and without the cache
    monkeypatch.setenv("PCDM_LAYOUT", "ragged")
    cfg = I.InstanceConfig("zr", 20_000, 8_000, 12, 300, rows="zipf")
    inst = I.generate(cfg, seed=1)
    for cache in ("0", "1"):
        monkeypatch.setenv("PCDM_HOT_CACHE", cache)
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 2048, 60, seed=2,
                       variant="packed")
        assert out["stats"]["lanes_per_column"] == 0
        assert_parity(out)
        _check_r(out)


def test_ragged_logistic(gpu, monkeypatch):
    monkeypatch.setenv("PCDM_LAYOUT", "ragged")
    m, n = 3000, 2000
    lens = np.random.default_rng(3).integers(1, 90, size=n)
    c, r, v = I.random_csc(m, n, lens, seed=3)
    y = torch.where(torch.randn(m, generator=torch.Generator().manual_seed(4)) >= 0, 1.0, -1.0)
    lam = 0.5
    res = oracle.logistic_run(m, c.numpy(), r.numpy(), v.numpy(), y.numpy(), lam, 128, 150, 1)
    F_orc = oracle.logistic_objective(m, c.numpy(), r.numpy(), v.numpy(), y.numpy(), lam, res.x)
    with pcdm.Problem(m, n, c.to(gpu), r.to(gpu), v.to(gpu), y.to(gpu), lam, loss="logistic") as prob:
        x = torch.zeros(n, device=gpu)
        prob.run(x, 128, 150, seed=1, variant="packed")
        assert prob.stats()["lanes_per_column"] == 0
        assert abs(prob.objective(x) - F_orc) <= 1e-5 * abs(F_orc)
        assert np.max(np.abs(to_host(x) - res.x)) <= 1e-4 * np.max(np.abs(res.x))
