"""One short tiny-config run per iteration loop, for compute-sanitizer (memcheck,
racecheck, synccheck): the loops that rely on the hand-rolled grid barrier (grid,
packed), shared-memory staging (smem) and the batched passes (screened and
grid-barrier step pass).  Checks the result against the oracle too.

    compute-sanitizer --tool racecheck python tools/sanitize_tiny.py [variant ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1212_0873_b200 import instances as I  # noqa: E402
from paper_1212_0873_b200 import pcdm  # noqa: E402


def main(variants):
    dev = torch.device("cuda:0")
    inst = I.generate("tiny", seed=0)
    c, r, v, b = inst.numpy()
    tau, iters = 32, 60
    res = oracle.run(inst.m, c, r, v, b, inst.lam, tau, iters, 0)
    Fo = oracle.objective(inst.m, c, r, v, b, inst.lam, res.x)
    with pcdm.Problem.from_instance(inst.to(dev)) as prob:
        for variant in variants:
            x = torch.zeros(inst.n, dtype=torch.float32, device=dev)
            prob.run(x, tau, iters, seed=0, variant=variant)
            F = prob.objective(x)
            ok = abs(F - Fo) <= 1e-5 * abs(Fo)
            print("sanitize %-8s F_gpu=%.9g F_oracle=%.9g %s" % (variant, F, Fo, "OK" if ok else "MISMATCH"))
            assert ok


if __name__ == "__main__":
    main(sys.argv[1:] or ["smem", "grid", "packed", "batched"])
