"""Full-length parity: the CUDA path against the oracle over the whole run each
benchmarked config times (alg:PCD1 is a K-iteration trajectory, PAPER.md:177-186;
K from BASELINE.json's configs):

  huge    m = 1e8, n = 5e8, 5e9 nonzeros, tau = 2^18, all 500 iterations, in the
          launch configuration bench.py times (AUTO -> the batched loop) and on
          the packed loop; the oracle runs on the sub-matrix of the columns
          S_0..S_499 touch (with x_0 = 0 no other column can move) and omega
          counted over the full matrix;
  large   m = 2e6, n = 1e7, 2e8 nonzeros, tau = 65536, all 2000 iterations;
  skewed  Zipf(1.1) rows, m = n = 1e6, tau in {2^8, 2^12, 2^16}, all 10^4
          iterations each.

Bar (north_star): sample sets and omega bit-exact, |F_gpu - F_orc| <= 1e-5 |F_orc|,
||x_gpu - x_orc||_inf <= 1e-4 ||x_orc||_inf.  The oracle runs were started in
background processes by the `gpu` fixture (tests/fullrun_jobs.py) and these
tests run last."""
import numpy as np
import pytest
import torch

import fullrun_jobs as J
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import F_RTOL, X_RTOL, to_host

pytestmark = [pytest.mark.gpu, pytest.mark.fullrun]


def _check(tag, F_gpu, xg, res, r_gpu=None):
    F_orc = float(res["F"])
    assert abs(F_gpu - F_orc) <= F_RTOL * abs(F_orc), (tag, F_gpu, F_orc)
    xo = res["x"]
    scale = max(float(np.max(np.abs(xo))), 1e-30)
    dx = float(np.max(np.abs(xg.astype(np.float64) - xo)))
    assert dx <= X_RTOL * scale, (tag, dx, scale)
    if r_gpu is not None:
        ro = res["r"]
        assert float(np.max(np.abs(r_gpu.astype(np.float64) - ro))) <= 1e-4 * float(np.max(np.abs(ro))), tag
    print("%s: F_gpu=%.10g F_orc=%.10g relF=%.2e dx_rel=%.2e (oracle loop %.1f s)"
          % (tag, F_gpu, F_orc, abs(F_gpu - F_orc) / abs(F_orc), dx / scale, float(res["loop_seconds"])))


def _run(prob, inst, tau, iters, variant="auto"):
    dev = inst.colptr.device
    x = torch.zeros(inst.n, dtype=torch.float32, device=dev)
    prob.run(x, tau, iters, seed=0, variant=variant)
    st = prob.stats()
    assert st["iters"] == iters
    r = torch.empty(inst.m, dtype=torch.float32, device=dev)
    prob.residual(r)
    return prob.objective(x), x, to_host(r), st


@pytest.mark.parametrize("tau", J.SKEWED_TAUS)
def test_fullrun_skewed(gpu, tau):
    inst = I.generate("skewed", seed=0, device=gpu)
    with pcdm.Problem.from_instance(inst) as prob:
        F, x, r, st = _run(prob, inst, tau, J.SKEWED_ITERS)
        res = J.get("skewed_%d" % tau).result()
        assert prob.omega == int(res["omega"])
        _check("skewed tau=%d (%s)" % (tau, st["variant"]), F, to_host(x), res, r)


def test_fullrun_large(gpu):
    cfg = I.CONFIGS["large"]
    inst = I.generate(cfg, seed=0, device=gpu)
    with pcdm.Problem.from_instance(inst) as prob:
        F, x, r, st = _run(prob, inst, cfg.tau, J.LARGE_ITERS)
        res = J.get("large").result()
        assert prob.omega == int(res["omega"])
        _check("large (%s)" % st["variant"], F, to_host(x), res, r)


def test_fullrun_huge(gpu):
    cfg = I.CONFIGS["huge"]
    if torch.cuda.get_device_properties(gpu).total_memory < 150e9:
        pytest.skip("the huge config needs ~120 GB of device memory")
    inst = I.generate(cfg, seed=0, device=gpu)
    prob = pcdm.Problem.from_instance(inst)
    # sample sets of S_0, S_1, S_250, S_499 at the huge shape, bit for bit
    want = np.load(J.slots_path("huge"))
    got = torch.empty(cfg.tau, dtype=torch.int32, device=gpu)
    for t, k in enumerate((0, 1, J.HUGE_ITERS // 2, J.HUGE_ITERS - 1)):
        pcdm.pcdm_sample(cfg.n, cfg.tau, 0, k, 1, got)
        assert np.array_equal(to_host(got), want[t]), k
    del inst.rowidx, inst.val
    torch.cuda.empty_cache()
    runs = {}
    for variant, name in (("auto", "batched"), ("packed", "packed")):
        F, x, r, st = _run(prob, inst, cfg.tau, J.HUGE_ITERS, variant)
        assert st["variant"] == pcdm.VARIANTS[name]
        runs[name] = (F, to_host(x), r)
        del x
    omega_gpu = prob.omega
    prob.close()
    res = J.get("huge").result()
    assert omega_gpu == int(res["omega_full"])  # bit-exact over all 5e9 entries
    cols = res["cols"]
    for name, (F, xg, r) in runs.items():
        untouched = np.ones(xg.size, dtype=bool)
        untouched[cols] = False
        assert not np.any(xg[untouched]), name
        _check("huge %s" % name, F, xg[cols], res, r)
