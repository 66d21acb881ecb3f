"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bit-exact: Philox words, sampled slot arrays, omega, row histogram.
Tolerance (north_star, BASELINE.json): F within 1e-5 relative, ||dx||_inf <=
1e-4 ||x||_inf; L_i within fp32 rounding of the oracle's fp64 value.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import ref_sampler
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import assert_parity, run_both, to_host

pytestmark = pytest.mark.gpu


# ------------------------------------------------------------------ Philox / sampler
def test_philox_matches_oracle_and_curand(gpu):
    rng = np.random.default_rng(0)
    N = 4096
    ctr = rng.integers(0, 1 << 32, size=4 * N, dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 1 << 32, size=2 * N, dtype=np.uint64).astype(np.uint32)
    out = np.zeros(4 * N, dtype=np.uint32)
    pcdm.pcdm_philox(ctr, key, out, stream=0)
    for t in range(0, N, 97):
        assert list(out[4 * t:4 * t + 4]) == list(oracle.philox4x32_10(ctr[4 * t:4 * t + 4], key[2 * t:2 * t + 2]))
    # P1: the device generator against cuRAND's curand_Philox4x32_10 on 1e6 pairs
    assert pcdm.pcdm_philox_check_curand(1 << 20, 12345) == 0


@pytest.mark.parametrize("n,tau,count", [
    (1, 1, 3), (2, 1, 5), (2, 2, 2), (5, 2, 50), (7, 5, 50), (20, 8, 50), (20, 15, 30),
    (100, 50, 20), (100, 51, 20), (97, 96, 10), (64, 64, 3), (1000, 32, 200),
    (100_000, 1024, 100), (3000, 1400, 5)])
def test_sampler_bitexact_small(gpu, n, tau, count):
    for seed in (0, 7):
        for first in (0, 1000):
            got = np.zeros(count * tau, dtype=np.int32)
            pcdm.pcdm_sample(n, tau, seed, first, count, got, stream=0)
            got = got.reshape(count, tau)
            for k in range(count):
                want = oracle.sample(seed, first + k, tau, n)
                assert np.array_equal(got[k], want), (seed, first + k)
            if n * count <= 4000:
                assert list(got[0]) == ref_sampler.sample(seed, first, tau, n)


@pytest.mark.parametrize("cfg,tau,count", [("skewed", 1 << 16, 12), ("skewed", 1 << 8, 50),
                                           ("large", 65536, 8), ("huge", 1 << 18, 3)])
def test_sampler_bitexact_config_shapes(gpu, cfg, tau, count):
    n = I.CONFIGS[cfg].n
    got = torch.zeros(count * tau, dtype=torch.int32, device=gpu)
    pcdm.pcdm_sample(n, tau, 0, 0, count, got)
    got = to_host(got).reshape(count, tau)
    for k in range(count):
        assert np.array_equal(got[k], oracle.sample(0, k, tau, n)), k


@pytest.mark.parametrize("n,tau,count", [(9000, 4400, 4), (8193, 4096, 3), (1 << 20, 1 << 17, 3), (50000, 4096, 20)])
def test_sampler_bitexact_large_tau(gpu, n, tau, count):
    # larger tau, and n close to 2 tau (many ownership rounds), over several iterations
    for seed in (0, 5):
        got = np.zeros(count * tau, dtype=np.int32)
        pcdm.pcdm_sample(n, tau, seed, 77, count, got, stream=0)
        for k in range(count):
            assert np.array_equal(got[k * tau:(k + 1) * tau], oracle.sample(seed, 77 + k, tau, n)), (seed, k)


def test_sampler_high_collision_rounds(gpu):
    # tau close to n/2 forces many ownership rounds; still bit-exact
    n, tau, count = 4001, 2000, 6
    got = np.zeros(count * tau, dtype=np.int32)
    pcdm.pcdm_sample(n, tau, 3, 0, count, got, stream=0)
    for k in range(count):
        assert np.array_equal(got[k * tau:(k + 1) * tau], oracle.sample(3, k, tau, n))


# ------------------------------------------------------------------ omega, L, histogram
@pytest.mark.parametrize("cfg", ["tiny", "medium", "skewed"])
def test_omega_L_counts(gpu, cfg):
    inst = I.generate(cfg, seed=0, device=gpu)
    prob = pcdm.Problem.from_instance(inst)
    c, r, v, b = inst.numpy()
    assert prob.omega == oracle.omega(inst.m, r)
    counts = torch.zeros(inst.m, dtype=torch.int32, device=gpu)
    prob.row_counts(counts)
    assert np.array_equal(to_host(counts), oracle.row_counts(inst.m, r))
    L = torch.zeros(inst.n, dtype=torch.float32, device=gpu)
    prob.col_norms(L)
    Lo = oracle.col_norms(c, v).astype(np.float32)  # fp64 value rounded to fp32
    np.testing.assert_allclose(to_host(L), Lo, rtol=2e-7, atol=0)
    prob.close()


@pytest.mark.parametrize("hot_count", [255, 256])
def test_row_counts_byte_counters_and_fallback(gpu, hot_count):
    # m > 2^26: two passes of byte counters (rows [0, 2^26) and [2^26, m)); a row stored
    # 255 times stays on them, 256 times overflows a byte and the 32-bit passes recount
    m, n, per = (1 << 26) + 4099, 2000, 40
    rng = np.random.default_rng(11)
    hot = (1 << 26) + 3
    cols = []
    for i in range(n):
        rows = np.unique(rng.integers(0, m, size=per))
        extra = [m - 1, (1 << 26) - 1, 1 << 26] if i % 7 == 0 else []
        if i < hot_count:
            extra.append(hot)
        cols.append(np.unique(np.concatenate([rows, np.array(extra, dtype=np.int64)])))
    lens = np.array([len(c) for c in cols])
    colptr = np.zeros(n + 1, dtype=np.int64)
    colptr[1:] = np.cumsum(lens)
    rowidx = np.concatenate(cols).astype(np.int32)
    val = rng.normal(size=rowidx.size).astype(np.float32)
    b = np.zeros(m, dtype=np.float32)
    dev = gpu
    prob = pcdm.Problem(m, n, torch.as_tensor(colptr, device=dev), torch.as_tensor(rowidx, device=dev),
                        torch.as_tensor(val, device=dev), torch.as_tensor(b, device=dev), 0.1)
    counts_o = oracle.row_counts(m, rowidx)
    assert counts_o[hot] == hot_count
    assert prob.omega == oracle.omega(m, rowidx) == int(counts_o.max())
    counts = torch.zeros(m, dtype=torch.int32, device=dev)
    prob.row_counts(counts)
    assert np.array_equal(to_host(counts), counts_o)
    L = torch.zeros(n, dtype=torch.float32, device=dev)
    prob.col_norms(L)
    np.testing.assert_allclose(to_host(L), oracle.col_norms(colptr, val).astype(np.float32), rtol=2e-7, atol=0)
    prob.close()


# ------------------------------------------------------------------ full runs
@pytest.mark.parametrize("variant", ["auto", "smem", "block", "grid"])
def test_tiny_config_full_run(gpu, variant):
    # BASELINE configs[0]: tiny, tau = 32, 2000 iterations, seed 0
    inst = I.generate("tiny", seed=0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 32, 2000, seed=0,
                   variant=variant)
    assert_parity(out)
    assert out["stats"]["iters"] == 2000
    assert out["F_orc"] < 0.5 * float((inst.b.double() ** 2).sum())


@pytest.mark.parametrize("form", [("1", "1"), ("1", "2"), ("1", "4"), ("1", "8"), ("1", "16"), ("1", "32"), ("0", "16")])
def test_smem_one_barrier_kernel(gpu, monkeypatch, form):
    # the shared-memory loop: the one-barrier kernel (double-buffered r, the previous
    # step replayed from its column) with E = 12, 6, 3, 2, 1, 1 entries per lane, and the
    # two-barrier list kernel (PCDM_SMEM1=0); full tiny run, then a nonzero start with
    # a refresh after every 3rd iteration (the replay is dropped at each refresh)
    monkeypatch.setenv("PCDM_SMEM1", form[0])
    monkeypatch.setenv("PCDM_SMEM_LANES", form[1])
    inst = I.generate("tiny", seed=0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 32, 2000, seed=0,
                   variant="smem")
    assert_parity(out)
    c, r, v, b, lam = _ragged(600, 250, np.random.default_rng(3).integers(0, 13, size=250), 8)
    for tau in (1, 5, 64):
        out = run_both(c, r, v, b, lam, 600, tau, 90, seed=tau, variant="smem", refresh_every=3,
                       x0=np.random.default_rng(5).normal(size=250))
        assert_parity(out)
        assert out["stats"]["refreshes"] == 30
        np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0, atol=1e-4 * np.max(np.abs(out["res"].r)))


def test_medium_config_full_run(gpu):
    inst = I.generate("medium", seed=0)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 1024, 10_000, seed=0,
                   variant="packed")
    assert_parity(out)
    assert out["stats"]["variant"] == pcdm.VARIANTS["packed"]


@pytest.mark.parametrize("tau", [1 << 8, 1 << 12, 1 << 16])
def test_skewed_config(gpu, tau):
    inst = I.generate("skewed", seed=0)
    iters = {1 << 8: 3000, 1 << 12: 1000, 1 << 16: 100}[tau]
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, tau, iters, seed=0)
    assert_parity(out)


def test_large_config_reduced_iters(gpu):
    inst = I.generate("large", seed=0, device=gpu)
    out = run_both(inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, inst.m, 65536, 40, seed=0)
    assert_parity(out)


# ------------------------------------------------------------------ edge cases
def _ragged(m, n, lens, seed, lam_frac=0.1):
    colptr, rowidx, val = I.random_csc(m, n, lens, seed=seed)
    b = I.random_b(m, seed=seed)
    return colptr, rowidx, val, b, I.lam_for(colptr, rowidx, val, b, lam_frac)


@pytest.mark.parametrize("variant", ["smem", "block", "grid", "packed", "auto"])
def test_ragged_columns_with_empty_and_long(gpu, variant):
    m, n = 3000, 700
    rng = np.random.default_rng(1)
    lens = rng.integers(0, 40, size=n)
    lens[:7] = 0
    lens[10] = 2999
    lens[11] = 700
    c, r, v, b, lam = _ragged(m, n, lens, 4)
    for tau in (1, 7, 300, 699, 700):
        out = run_both(c, r, v, b, lam, m, tau, 60, seed=tau, variant=variant,
                       x0=np.random.default_rng(2).normal(size=n) * (np.arange(n) % 5 == 0))
        assert_parity(out)


@pytest.mark.parametrize("variant", ["smem", "grid"])
def test_lambda_zero_and_beta_override(gpu, variant):
    c, r, v, b, lam = _ragged(400, 300, np.full(300, 6), 9)
    assert_parity(run_both(c, r, v, b, 0.0, 400, 16, 300, seed=1, variant=variant))
    assert_parity(run_both(c, r, v, b, lam, 400, 16, 300, seed=1, beta_override=3.5, variant=variant))


def test_resume_continues_the_stream(gpu):
    c, r, v, b, lam = _ragged(2000, 1500, np.full(1500, 8), 5)
    dev = gpu
    prob = pcdm.Problem(2000, 1500, c.to(dev), r.to(dev), v.to(dev), b.to(dev), lam)
    x1 = torch.zeros(1500, device=dev)
    prob.run(x1, 64, 300, seed=11, refresh_every=-1)
    x2 = torch.zeros(1500, device=dev)
    prob.run(x2, 64, 120, seed=11, refresh_every=-1)
    prob.run(x2, 64, 180, seed=11, first_iter=120, refresh_every=-1)
    xo = oracle.run(2000, to_host(c), to_host(r), to_host(v), to_host(b), lam, 64, 300, 11,
                    refresh_every=-1).x
    for x in (x1, x2):
        assert np.max(np.abs(to_host(x) - xo)) <= 1e-4 * np.max(np.abs(xo))
    prob.close()


def test_host_and_device_x_agree(gpu):
    inst = I.generate("tiny", seed=3)
    prob = pcdm.Problem.from_instance(inst.to(gpu))
    xh = np.zeros(inst.n, dtype=np.float32)
    xd = torch.zeros(inst.n, dtype=torch.float32, device=gpu)
    prob.run(xh, 32, 500, seed=2, variant="grid")
    prob.run(xd, 32, 500, seed=2, variant="grid")
    np.testing.assert_allclose(xh, to_host(xd), rtol=1e-5, atol=1e-6)
    assert abs(prob.objective(xh) - prob.objective(xd)) <= 1e-6 * prob.objective(xd)
    prob.close()


@pytest.mark.parametrize("refresh", [-1, 1, 7])
@pytest.mark.parametrize("variant", ["grid", "smem"])
def test_refresh_cadence(gpu, refresh, variant):
    # (the shared-memory variant refreshes inside its kernel, the others between launches)
    c, r, v, b, lam = _ragged(500, 400, np.full(400, 5), 6)
    out = run_both(c, r, v, b, lam, 500, 40, 100, seed=4, refresh_every=refresh, variant=variant)
    assert_parity(out)
    assert out["stats"]["refreshes"] == (0 if refresh < 0 else 100 // refresh)
    # maintained residual vs the oracle's (and vs Ax-b of the oracle's x)
    np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0, atol=1e-4 * np.max(np.abs(out["res"].r)))


def test_objective_matches_oracle(gpu):
    inst = I.generate("medium", seed=1)
    x = torch.randn(inst.n, generator=torch.Generator().manual_seed(0)) * (torch.rand(inst.n) < 0.05)
    prob = pcdm.Problem.from_instance(inst.to(gpu))
    F = prob.objective(x.to(gpu))
    c, r, v, b = inst.numpy()
    Fo = oracle.objective(inst.m, c, r, v, b, inst.lam, x.numpy().astype(np.float64))
    assert abs(F - Fo) <= 1e-12 * abs(Fo)
    prob.close()


# ------------------------------------------------------------------ errors
def test_errors(gpu):
    c, r, v, b, lam = _ragged(50, 40, np.full(40, 3), 1)
    dev = gpu
    bad_r = r.clone()
    bad_r[5] = 50
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.Problem(50, 40, c.to(dev), bad_r.to(dev), v.to(dev), b.to(dev), lam)
    assert e.value.status == pcdm.PCDM_EINVAL and "row index" in e.value.message
    unsorted = r.clone()
    unsorted[0], unsorted[1] = r[1], r[0]
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.Problem(50, 40, c.to(dev), unsorted.to(dev), v.to(dev), b.to(dev), lam)
    assert "strictly increasing" in e.value.message
    bad_c = c.clone()
    bad_c[-1] += 1
    with pytest.raises(pcdm.PCDMError):
        pcdm.Problem(50, 40, bad_c.to(dev), r.to(dev), v.to(dev), b.to(dev), lam)
    nan_v = v.clone()
    nan_v[3] = float("nan")
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.Problem(50, 40, c.to(dev), r.to(dev), nan_v.to(dev), b.to(dev), lam)
    assert "val" in e.value.message
    prob = pcdm.Problem(50, 40, c.to(dev), r.to(dev), v.to(dev), b.to(dev), lam)
    x = torch.zeros(40, device=dev)
    for tau in (0, 41):
        with pytest.raises(pcdm.PCDMError) as e:
            prob.run(x, tau, 1)
        assert e.value.status == pcdm.PCDM_EINVAL
    x[3] = float("inf")
    with pytest.raises(pcdm.PCDMError) as e:
        prob.run(x, 4, 1)
    assert e.value.status == pcdm.PCDM_EINVAL
    x = torch.zeros(40, device=dev)
    with pytest.raises(pcdm.PCDMError) as e:
        prob.run(x, 40, 200, beta_override=1e-30, variant="grid")
    assert e.value.status == pcdm.PCDM_EDIVERGED
    prob.close()


# ------------------------------------------------------------------ packed-block loop
@pytest.mark.parametrize("one_barrier", ["0", "1"])
@pytest.mark.parametrize("lens_kind", ["uniform10", "uniform20", "ragged"])
def test_packed_variant_both_barrier_schemes(gpu, monkeypatch, one_barrier, lens_kind):
    monkeypatch.setenv("PCDM_ONE_BARRIER", one_barrier)
    m, n = 5000, 4000
    rng = np.random.default_rng(3)
    lens = {"uniform10": np.full(n, 10), "uniform20": np.full(n, 20),
            "ragged": rng.integers(0, 62, size=n)}[lens_kind]
    if lens_kind == "ragged":
        lens[:5] = 0
        lens[5] = 62
    c, r, v, b, lam = _ragged(m, n, lens, 8, lam_frac=0.05)
    x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 7 == 0)
    for tau, iters, refresh in ((1, 300, 0), (64, 200, 0), (1000, 40, 7), (4000, 5, -1)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="packed", x0=x0,
                       refresh_every=refresh)
        assert out["stats"]["variant"] == pcdm.VARIANTS["packed"]
        assert_parity(out)
        np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0,
                                   atol=1e-4 * np.max(np.abs(out["res"].r)))


@pytest.mark.parametrize("iter_chunk", ["3", "64"], ids=["3-iteration-launches", "long-launches"])
@pytest.mark.parametrize("reg_replay", ["1", "0"], ids=["register-replay", "list-replay"])
def test_packed_one_slot_per_group(gpu, monkeypatch, reg_replay, iter_chunk):
    # a grid that covers tau in one round: the previous iteration's step is replayed from
    # the registers of the group that took it (pcdm_packed1_kernel, no step lists), both
    # residual buffers equal at every launch boundary (3-iteration launches flip the
    # buffer parity from launch to launch); the list-based loop on the same runs;
    # dense nonzero starts (many steps per iteration), refreshes, idle slots
    monkeypatch.setenv("PCDM_REG_REPLAY", reg_replay)
    monkeypatch.setenv("PCDM_ITER_CHUNK", iter_chunk)
    m, n = 5000, 4000
    rng = np.random.default_rng(13)
    lens = rng.integers(0, 30, size=n)
    c, r, v, b, lam = _ragged(m, n, lens, 9, lam_frac=0.05)
    x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 3 == 0)
    nz = {}
    for tau, iters, refresh, sampling in ((1, 200, 0, None), (64, 203, 0, None), (1000, 41, 7, None),
                                          (4000, 6, -1, None), (700, 60, 0, ("binomial", 700, 0.6, None))):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="packed", x0=x0,
                       refresh_every=refresh, sampling=sampling)
        assert out["stats"]["variant"] == pcdm.VARIANTS["packed"]
        assert_parity(out)
        np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0,
                                   atol=1e-4 * np.max(np.abs(out["res"].r)))
        nz[tau] = out["stats"]["nonzero_deltas"]
    assert nz[1000] > 1000 and nz[64] > 0  # the step count survives the register form


@pytest.mark.parametrize("iter_chunk", ["3", "64"], ids=["3-iteration-launches", "long-launches"])
@pytest.mark.parametrize("local", ["1", "0"], ids=["cta-local-replay", "global-lists"])
def test_packed_cta_local_replay(gpu, monkeypatch, local, iter_chunk):
    # several slots per group (tau above the grid's groups) and one slot per group with
    # the register form off: each CTA keeps its steps in shared-memory lists and replays
    # them itself (no global step lists; both residual buffers equal at launch end),
    # against the global-list loop on the same runs; dense nonzero starts, refreshes
    monkeypatch.setenv("PCDM_LOCAL_REPLAY", local)
    monkeypatch.setenv("PCDM_REG_REPLAY", "0")
    monkeypatch.setenv("PCDM_ITER_CHUNK", iter_chunk)
    m, n = 6000, 40_000
    c, r, v, b, lam = _ragged(m, n, np.random.default_rng(2).integers(0, 14, size=n), 23, lam_frac=0.05)
    x0 = np.random.default_rng(6).normal(size=n) * (np.arange(n) % 5 == 0)
    for tau, iters, refresh in ((40_000, 7, 3), (30_000, 13, 0), (999, 41, 0), (64, 100, 7)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="packed", x0=x0, refresh_every=refresh)
        assert out["stats"]["variant"] == pcdm.VARIANTS["packed"]
        assert_parity(out)
        np.testing.assert_allclose(out["r_gpu"], out["res"].r, rtol=0,
                                   atol=1e-4 * np.max(np.abs(out["res"].r)))
        assert out["stats"]["nonzero_deltas"] > 0


def test_long_columns_take_the_ragged_layout(gpu):
    # a column over 62 entries: the packed loop runs on the ragged layout (a CTA for the
    # long column, sub-warps for the rest); the uniform-only loops are rejected
    c, r, v, b, lam = _ragged(300, 20, [100] + [3] * 19, 2)
    prob = pcdm.Problem(300, 20, c.to(gpu), r.to(gpu), v.to(gpu), b.to(gpu), lam)
    prob.run(torch.zeros(20, device=gpu), 4, 1, variant="packed")
    assert prob.stats()["lanes_per_column"] == 0
    with pytest.raises(pcdm.PCDMError) as e:
        prob.run(torch.zeros(20, device=gpu), 4, 1, variant="batched")
    assert e.value.status == pcdm.PCDM_EINVAL
    prob.run(torch.zeros(20, device=gpu), 4, 1)  # AUTO
    prob.close()
    assert_parity(run_both(c, r, v, b, lam, 300, 4, 50, seed=1, variant="packed"))


# ------------------------------------------------------------------ many launches per run
@pytest.mark.parametrize("presample", ["1", "0"], ids=["presampled", "in-stream"])
@pytest.mark.parametrize("iter_chunk", ["3", "16"], ids=["launch-per-sampler-chunk", "launch-spans-chunks"])
@pytest.mark.parametrize("variant", ["packed", "grid", "batched"])
def test_many_chunks_per_run(gpu, monkeypatch, variant, iter_chunk, presample):
    # small sampler chunks force many sampler passes per run; iteration-kernel launches
    # of 3 iterations, or of 16 whose slots come from several sampler chunks; the slots
    # presampled on the side stream (each launch waiting on its own pass's event) or
    # drawn in the run's stream window by window
    monkeypatch.setenv("PCDM_CHUNK", "3")
    monkeypatch.setenv("PCDM_ITER_CHUNK", iter_chunk)
    monkeypatch.setenv("PCDM_BATCHED_CHUNK", iter_chunk)
    monkeypatch.setenv("PCDM_PRESAMPLE_DEV", presample)
    c, r, v, b, lam = _ragged(3000, 2500, np.full(2500, 12), 12)
    for tau, iters, refresh in ((256, 61, 0), (2500, 7, 4), (33, 200, -1)):
        out = run_both(c, r, v, b, lam, 3000, tau, iters, seed=5, variant=variant, refresh_every=refresh)
        assert_parity(out)
        assert out["stats"]["iter_launches"] >= iters // int(iter_chunk)


# ------------------------------------------------------------------ other DU samplings (NEXT-1)
SAMPLINGS = [("independent", 37, 1.0, None), ("independent", 700, 1.0, None), ("binomial", 64, 0.3, None),
             ("binomial", 700, 0.75, None), ("binomial", 500, 1.0, None),
             ("du", 40, 1.0, list(np.random.default_rng(9).dirichlet(np.ones(41))))]


@pytest.mark.parametrize("spec", SAMPLINGS, ids=lambda s: "%s-%d" % (s[0], s[1]))
def test_sampling_slot_arrays_bitexact(gpu, spec):
    n = 700
    count = 12
    got = np.zeros(count * spec[1], dtype=np.int32)
    pcdm.pcdm_sample_sampling(n, pcdm.Sampling(*spec), 5, 3, count, got, stream=0)
    got = got.reshape(count, spec[1])
    osp = oracle.Sampling(*spec)
    for k in range(count):
        assert np.array_equal(got[k], oracle.sample_kind(osp, 5, 3 + k, n)), k
    # huge-shaped independent / binomial draws too
    for spec2 in (("independent", 1 << 16, 1.0, None), ("binomial", 1 << 16, 0.5, None)):
        g = torch.zeros(2 << 16, dtype=torch.int32, device=gpu)
        pcdm.pcdm_sample_sampling(500_000_000, pcdm.Sampling(*spec2), 1, 0, 2, g)
        g = to_host(g).reshape(2, -1)
        for k in range(2):
            assert np.array_equal(g[k], oracle.sample_kind(oracle.Sampling(*spec2), 1, k, 500_000_000))


@pytest.mark.parametrize("spec", SAMPLINGS, ids=lambda s: "%s-%d" % (s[0], s[1]))
@pytest.mark.parametrize("variant", ["packed", "grid", "smem"])
def test_sampling_runs_match_oracle(gpu, spec, variant):
    m, n = 900, 700
    c, r, v, b, lam = _ragged(m, n, np.random.default_rng(2).integers(1, 30, size=n), 31)
    out = run_both(c, r, v, b, lam, m, spec[1], 120, seed=4, variant=variant, sampling=spec)
    assert_parity(out)
    assert out["beta_gpu"] == pytest.approx(out["res"].beta, rel=1e-12)


def test_sampling_errors(gpu):
    c, r, v, b, lam = _ragged(50, 40, np.full(40, 3), 1)
    prob = pcdm.Problem(50, 40, c.to(gpu), r.to(gpu), v.to(gpu), b.to(gpu), lam)
    x = torch.zeros(40, device=gpu)
    for bad in (pcdm.Sampling("binomial", 8, p_b=0.0), pcdm.Sampling("binomial", 8, p_b=1.5),
                pcdm.Sampling("du", 4, q=[0.5, 0.5, 0.5, 0.0, 0.0]), pcdm.Sampling("du", 30, q=np.full(31, 1 / 31)),
                pcdm.Sampling("independent", 41)):
        with pytest.raises(pcdm.PCDMError) as e:
            prob.run(x, 0, 1, sampling=bad)
        assert e.value.status == pcdm.PCDM_EINVAL
    prob.close()


# ------------------------------------------------------------------ x in the block headers (packed loop)
@pytest.mark.parametrize("mode", [("1", None), ("0", None), ("1", "5")], ids=["hdr", "array", "hdr-overflow"])
def test_x_in_block_headers(gpu, monkeypatch, mode):
    monkeypatch.setenv("PCDM_X_IN_BLOCK", mode[0])
    if mode[1]:
        monkeypatch.setenv("PCDM_XLIST_CAP", mode[1])  # tiny dirty list: start / end passes walk all columns
    m, n = 4000, 3000
    c, r, v, b, lam = _ragged(m, n, np.random.default_rng(4).integers(1, 40, size=n), 41)
    x0 = np.random.default_rng(5).normal(size=n) * (np.arange(n) % 3 == 0)
    for tau, iters, refresh in ((64, 150, 0), (1500, 30, 7), (3000, 6, -1)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="packed", x0=x0, refresh_every=refresh)
        assert_parity(out)


def test_caller_changes_x_between_runs(gpu):
    # the library must take the caller's x afresh at every run (headers are re-synchronised)
    m, n = 3000, 2000
    c, r, v, b, lam = _ragged(m, n, np.full(n, 12), 42)
    prob = pcdm.Problem(m, n, c.to(gpu), r.to(gpu), v.to(gpu), b.to(gpu), lam)
    x = torch.zeros(n, device=gpu)
    prob.run(x, 128, 200, seed=1, variant="packed")
    x1 = np.random.default_rng(6).normal(size=n) * (np.arange(n) % 5 == 1)
    x.copy_(torch.from_numpy(x1.astype(np.float32)))
    prob.run(x, 128, 100, seed=2, first_iter=200, variant="packed")
    xo = oracle.run(m, to_host(c), to_host(r), to_host(v), to_host(b), lam, 128, 100, 2, first_iter=200,
                    x0=x1.astype(np.float32).astype(np.float64)).x
    assert np.max(np.abs(to_host(x) - xo)) <= 1e-4 * np.max(np.abs(xo))
    # and a zero x after a run with a big support
    x.zero_()
    prob.run(x, 128, 50, seed=3, variant="packed")
    xo = oracle.run(m, to_host(c), to_host(r), to_host(v), to_host(b), lam, 128, 50, 3).x
    assert np.max(np.abs(to_host(x) - xo)) <= 1e-4 * np.max(np.abs(xo))
    prob.close()


# ------------------------------------------------------------------ host x: compact copy-back
@pytest.mark.parametrize("cap,refresh", [(None, 0), ("3", 0), (None, 9)], ids=["compact", "list-overflow", "refresh"])
def test_host_x_compact_copy_back(gpu, monkeypatch, cap, refresh):
    # packed loop with x in the block headers: only the dirty entries travel back to the host
    if cap:
        monkeypatch.setenv("PCDM_XLIST_CAP", cap)
    m, n = 6000, 20_000
    c, r, v, b, lam = _ragged(m, n, np.full(n, 8), 51, lam_frac=0.3)
    x0 = np.zeros(n, dtype=np.float32)
    x0[::997] = np.random.default_rng(7).normal(size=x0[::997].size).astype(np.float32)
    prob = pcdm.Problem(m, n, c.to(gpu), r.to(gpu), v.to(gpu), b.to(gpu), lam)
    xh = x0.copy()
    xd = torch.from_numpy(x0.copy()).to(gpu)
    prob.run(xh, 256, 40, seed=9, variant="packed", refresh_every=refresh)
    st = prob.stats()
    prob.run(xd, 256, 40, seed=9, variant="packed", refresh_every=refresh)
    np.testing.assert_allclose(xh, to_host(xd), rtol=1e-5, atol=1e-6)
    assert st["host_h2d_bytes"] == 4 * n
    if cap or refresh:  # an overflowed or restarted dirty list: the whole x travels back
        assert st["host_d2h_bytes"] == 4 * n
    else:
        assert 0 < st["host_d2h_bytes"] < 4 * n // 4
    xo = oracle.run(m, to_host(c), to_host(r), to_host(v), to_host(b), lam, 256, 40, 9,
                    x0=x0.astype(np.float64), refresh_every=refresh).x
    assert np.max(np.abs(xh - xo)) <= 1e-4 * np.max(np.abs(xo))
    prob.close()


# ------------------------------------------------------------------ dense-step bookkeeping on LASSO
@pytest.mark.parametrize("stage,dense", [("1", "0"), ("0", "1"), ("1", "1")])
def test_staged_step_list_and_dense_x(gpu, monkeypatch, stage, dense):
    # the logistic defaults (CTA-staged step lists, no dirty x list) forced on a LASSO
    # problem with many nonzero steps (lambda = 0), both barrier schemes, refreshes
    monkeypatch.setenv("PCDM_STAGE_LIST", stage)
    monkeypatch.setenv("PCDM_XLIST_DENSE", dense)
    m, n = 5000, 4000
    c, r, v, b, lam = _ragged(m, n, np.random.default_rng(9).integers(1, 30, size=n), 19)
    x0 = np.random.default_rng(4).normal(size=n) * (np.arange(n) % 5 == 0)
    for one_barrier in ("1", "0"):
        monkeypatch.setenv("PCDM_ONE_BARRIER", one_barrier)
        for tau, iters, refresh, lam_ in ((512, 120, 0, 0.0), (4000, 8, 3, lam), (64, 200, 0, lam)):
            out = run_both(c, r, v, b, lam_, m, tau, iters, seed=tau, variant="packed", x0=x0, refresh_every=refresh)
            assert_parity(out)
    # host x with a dense list: the whole x travels back
    prob = pcdm.Problem(m, n, c.to(gpu), r.to(gpu), v.to(gpu), b.to(gpu), 0.0)
    xh = np.zeros(n, dtype=np.float32)
    prob.run(xh, 512, 30, seed=1, variant="packed")
    assert prob.stats()["host_d2h_bytes"] == (4 * n if dense == "1" else prob.stats()["host_d2h_bytes"])
    xo = oracle.run(m, to_host(c), to_host(r), to_host(v), to_host(b), 0.0, 512, 30, 1).x
    assert np.max(np.abs(xh - xo)) <= 1e-4 * np.max(np.abs(xo))
    prob.close()


@pytest.mark.parametrize("pipeline", ["0", "1"])
def test_packed_slot_pipeline_on_and_off(gpu, monkeypatch, pipeline):
    # the software-pipelined slot loop (next block loaded before the current gathers) is
    # chosen for L2-resident r; both forms against the oracle, several slots per group
    monkeypatch.setenv("PCDM_PIPELINE", pipeline)
    m, n = 6000, 40_000
    c, r, v, b, lam = _ragged(m, n, np.random.default_rng(2).integers(0, 14, size=n), 23, lam_frac=0.05)
    x0 = np.random.default_rng(6).normal(size=n) * (np.arange(n) % 9 == 0)
    for tau, iters, refresh in ((40_000, 6, 3), (20_000, 12, 0), (999, 80, 0)):
        out = run_both(c, r, v, b, lam, m, tau, iters, seed=tau, variant="packed", x0=x0, refresh_every=refresh)
        assert_parity(out)
