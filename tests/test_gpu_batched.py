"""BATCHED variant (kernels_batched.cu): the same synchronous PCDM1 iteration
(alg:PCD1 PAPER.md:177-186, soft-threshold eq:h(x) PAPER.md:214-216) with the
partial derivatives computed as g_i = a_i^T r_0 + a_i^T (r_k - r_0) per chunk of
iterations.  Only the fp32 summation order of g_i changes, so the north_star
tolerances against the oracle apply unchanged: F within 1e-5 relative,
||dx||_inf <= 1e-4 ||x||_inf, and the maintained residual equals the oracle's."""
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


@pytest.mark.parametrize("lens_kind", ["uniform10", "uniform20", "ragged"])
def test_batched_matches_oracle(gpu, lens_kind):
    m, n = 5000, 4000
    rng = np.random.default_rng(3)
    lens = {"uniform10": np.full(n, 10), "uniform20": np.full(n, 20),
            "ragged": rng.integers(0, 62, size=n)}[lens_kind]
    if lens_kind == "ragged":
        lens[:5] = 0
        lens[5] = 62
    c, r, v, b, lam = _ragged(m, n, lens, 8, lam_frac=0.05)
    # a nonzero start: many nonzero steps per iteration, so many dirty rows per chunk
    x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 7 == 0)
    for tau, iters, refresh in ((1, 300, 0), (64, 200, 0), (1000, 40, 7), (4000, 5, -1)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="batched", x0=x0, refresh_every=refresh)
        assert out["stats"]["variant"] == pcdm.VARIANTS["batched"]
        assert_parity(out)
        _check_r(out)


def test_batched_tiny_and_medium_configs(gpu):
    inst = I.generate("tiny", seed=0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 32, 2000, seed=0, variant="batched")
    assert_parity(out)
    inst = I.generate("medium", seed=0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 1024, 2000, seed=0,
                   variant="batched")
    assert_parity(out)
    _check_r(out)


def test_batched_several_row_bins(gpu):
    # m > 2^21 rows: several row bins of the sweep; many columns sampled twice per chunk
    inst = I.generate(I.InstanceConfig("bins", 5_000_000, 300_000, 10, 3000, lam_frac=0.01), seed=1)
    x0 = np.random.default_rng(2).normal(size=inst.n) * (np.arange(inst.n) % 50 == 0)
    for tau, iters in ((65536, 30), (4096, 120)):
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=tau,
                       variant="batched", x0=x0)
        assert_parity(out)
        _check_r(out)


@pytest.mark.parametrize("chunk", ["1", "3"])
def test_batched_many_chunks(gpu, monkeypatch, chunk):
    monkeypatch.setenv("PCDM_CHUNK", chunk)
    c, r, v, b, lam = _ragged(3000, 2500, np.full(2500, 12), 12)
    for tau, iters, refresh in ((256, 61, 0), (2500, 7, 4), (33, 200, -1)):
        out = run_both(c, r, v, b, lam, 3000, tau, iters, seed=5, variant="batched", refresh_every=refresh)
        assert_parity(out)


SAMPLINGS = [("independent", 700, 1.0, None), ("binomial", 500, 0.6, None),
             ("du", 40, 1.0, list(np.random.default_rng(9).dirichlet(np.ones(41))))]


@pytest.mark.parametrize("spec", SAMPLINGS, ids=lambda s: "%s-%d" % (s[0], s[1]))
def test_batched_samplings(gpu, spec):
    c, r, v, b, lam = _ragged(3000, 2000, np.random.default_rng(1).integers(1, 25, size=2000), 3)
    out = run_both(c, r, v, b, lam, 3000, spec[1], 120, seed=4, variant="batched", sampling=spec)
    assert_parity(out)


@pytest.mark.parametrize("x_in_block", ["1", "0"])
def test_batched_x_storage_and_hot_rows(gpu, monkeypatch, x_in_block):
    monkeypatch.setenv("PCDM_X_IN_BLOCK", x_in_block)
    inst = I.generate(I.InstanceConfig("zipf_small", 20_000, 20_000, 20, 200, rows="zipf"), seed=0)
    for tau, iters in ((2048, 60), (200, 200)):
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=tau,
                       variant="batched")
        assert_parity(out)
        _check_r(out)


def test_batched_logistic(gpu):
    colptr, rowidx, val, y, lam = I.generate_logistic("logistic_small", seed=0)
    out = run_both_logistic(colptr, rowidx, val, y, lam, 20_000, 1024, 300, variant="batched")
    check(out)
    m, n = 600, 400
    lens = np.random.default_rng(5).integers(0, 20, size=n)
    lens[:3] = 0
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=6)
    y = _labels(m, 7)
    x0 = np.random.default_rng(8).normal(size=n) * (np.arange(n) % 4 == 0)
    for tau, lam in ((37, 1.0), (400, 0.1)):
        check(run_both_logistic(colptr, rowidx, val, y, lam, m, tau, 80, seed=tau, variant="batched", x0=x0,
                                first_iter=3))


def _auto_batched(monkeypatch, chunk="5"):
    # the size rule (r > 2 x L2) off: PCDM_BATCHED=1 makes AUTO take the batched loop with
    # its packed fallback on any size; the guard reads the step count synchronously
    monkeypatch.setenv("PCDM_BATCHED", "1")
    monkeypatch.setenv("PCDM_BATCHED_SYNC_CHECK", "1")
    monkeypatch.setenv("PCDM_BATCHED_CHUNK", chunk)


def test_auto_batched_falls_back_on_dense_steps(gpu, monkeypatch):
    # small lambda and a dense start: most steps nonzero, more dirty rows per snapshot than
    # the filters hold -> the packed loop takes over after the first snapshot (at an odd
    # iteration: the one-barrier loop starts from r2 = r and empty step lists)
    _auto_batched(monkeypatch)
    inst = I.generate(I.InstanceConfig("dense_steps", 200_000, 20_000, 10, 20_000, lam_frac=0.001), seed=2)
    x0 = np.random.default_rng(4).normal(size=inst.n)
    for tau, iters, refresh in ((4000, 23, 0), (4000, 40, 12), (20_000, 9, -1)):
        out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=tau, x0=x0,
                       refresh_every=refresh)
        assert out["stats"]["variant"] == pcdm.VARIANTS["packed"]
        assert out["stats"]["iter_launches"] >= 2
        assert_parity(out)
        _check_r(out)


def test_auto_batched_keeps_sparse_steps(gpu, monkeypatch):
    # large lambda from x = 0: few nonzero steps, the batched loop runs the whole run
    _auto_batched(monkeypatch)
    inst = I.generate(I.InstanceConfig("sparse_steps", 200_000, 20_000, 10, 100, lam_frac=0.5), seed=3)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 2000, 37, seed=3)
    assert out["stats"]["variant"] == pcdm.VARIANTS["batched"]
    assert_parity(out)
    _check_r(out)


@pytest.mark.parametrize("chunk", ["4", "7"])
def test_auto_batched_forced_fallback(gpu, monkeypatch, chunk):
    # the hand-off itself on a multi-bin instance, at an even and an odd iteration
    _auto_batched(monkeypatch, chunk)
    monkeypatch.setenv("PCDM_BATCHED_FORCE_FALLBACK", "1")
    inst = I.generate(I.InstanceConfig("bins", 5_000_000, 300_000, 10, 3000, lam_frac=0.01), seed=1)
    x0 = np.random.default_rng(2).normal(size=inst.n) * (np.arange(inst.n) % 50 == 0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 4096, 30, seed=7, x0=x0)
    assert out["stats"]["variant"] == pcdm.VARIANTS["packed"]
    assert_parity(out)
    _check_r(out)


# The step pass of the batched loop: the screened form (default for LASSO: speculative
# steps from g0, a test pass, one fix-up CTA replaying the chunk over its items) against
# the grid-barrier form (PCDM_BATCHED_SCREEN=0) and against the screened form with tiny
# shared-memory maps (PCDM_SCREEN_SMALL=1: D spills to the dense buffer, the stepped-column
# set overflows, items are read from global memory, steps overflow the shared list).
@pytest.mark.parametrize("mode", ["screen", "grid", "small"])
def test_batched_step_pass_forms(gpu, monkeypatch, mode):
    if mode == "grid":
        monkeypatch.setenv("PCDM_BATCHED_SCREEN", "0")
    if mode == "small":
        monkeypatch.setenv("PCDM_SCREEN_SMALL", "1")
    m, n = 5000, 4000
    rng = np.random.default_rng(13)
    for lens in (np.full(n, 10), rng.integers(0, 15, size=n)):
        c, r, v, b, lam = _ragged(m, n, lens, 9, lam_frac=0.05)
        x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 5 == 0)
        for tau, iters, refresh in ((64, 150, 0), (1000, 40, 7), (4000, 6, -1)):
            out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau + 1, variant="batched", x0=x0,
                           refresh_every=refresh)
            assert out["stats"]["variant"] == pcdm.VARIANTS["batched"]
            assert_parity(out)
            _check_r(out)
            if mode != "grid" and tau == 1000:
                # dense start: flagged slots step, so the later-slot scans run
                assert out["stats"]["screen_misses"] > 0
            if mode == "grid":
                assert out["stats"]["screen_misses"] == 0


def test_batched_screen_sparse_steps_no_misses(gpu):
    # from x = 0 with a large lambda the speculative steps are (almost) all the steps
    inst = I.generate(I.InstanceConfig("sparse_steps", 200_000, 20_000, 10, 100, lam_frac=0.5), seed=3)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 2000, 37, seed=3, variant="batched")
    assert_parity(out)
    _check_r(out)
    assert out["stats"]["screen_misses"] <= 2
