"""Setup quantities at BASELINE.json's full `huge` size (m = 1e8, n = 5e8, 5e9
nonzeros): omega and the column norms against independent computations of their
definitions (a chunked bincount of the row indices; host fp64 sums).  The whole
500-iteration run is checked against the oracle in test_gpu_fullrun.py."""
import numpy as np
import pytest
import torch

import oracle
from paper_1212_0873_b200 import instances as I
from paper_1212_0873_b200 import pcdm
from parity_util import to_host

pytestmark = pytest.mark.gpu


def test_huge_full_size_setup(gpu):
    cfg = I.CONFIGS["huge"]
    if torch.cuda.get_device_properties(gpu).total_memory < 150e9:
        pytest.skip("the huge config needs ~120 GB of device memory")
    inst = I.generate(cfg, seed=0, device=gpu)
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

    beta = prob.beta(cfg.tau)
    assert abs(beta - oracle.beta(prob.omega, cfg.tau, inst.n)) <= 1e-15 * beta
    prob.close()
    # the 500-iteration runs themselves are checked against the oracle in test_gpu_fullrun.py
