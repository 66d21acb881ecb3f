"""A/B of the residual-scatter alternatives on the skewed (Zipf-row)
config: hot-row scatters straight to global memory (red.global.add.f32) vs staged in
shared memory per CTA (PCDM_HOT_STAGE), for LASSO (sparse steps) and the logistic loss
on the same matrix (every visited coordinate steps, so every iteration scatters into
the hot rows).  Prints one JSON line per (loss, tau, stage)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1212_0873_b200 import instances as I  # noqa: E402
from paper_1212_0873_b200 import pcdm  # noqa: E402


def timed(prob, n, tau, iters, reps=3):
    x = torch.zeros(n, device="cuda")
    prob.run(x, tau, iters, seed=0)  # warm-up
    ms = []
    for r in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        prob.run(x, tau, iters, seed=0, first_iter=(r + 1) * iters)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    st = prob.stats()
    return min(ms), st


def main():
    os.environ["PCDM_DEBUG_KNOBS"] = "1"  # PCDM_HOT_STAGE is a debug knob
    pcdm.load()
    inst = I.generate("skewed", seed=0, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(5)
    y = torch.where(torch.randn(inst.m, generator=gen, device="cuda") >= 0, 1.0, -1.0)
    cases = [("lasso", 4096, 10000), ("lasso", 65536, 10000), ("logistic", 4096, 2000), ("logistic", 65536, 1000)]
    for loss, tau, iters in cases:
        for stage in ("0", "1"):
            os.environ["PCDM_HOT_STAGE"] = stage
            if loss == "lasso":
                prob = pcdm.Problem.from_instance(inst)
            else:
                prob = pcdm.Problem(inst.m, inst.n, inst.colptr, inst.rowidx, inst.val, y, 1.0, loss="logistic")
            ms, st = timed(prob, inst.n, tau, iters)
            print(json.dumps({"loss": loss, "tau": tau, "iters": iters, "hot_stage": int(stage), "ms": ms,
                              "updates_per_s": tau * iters / (ms / 1e3), "iter_kernel_ms": st["iter_kernel_ms"],
                              "hot_rows": st["hot_rows"], "nonzero_deltas": st["nonzero_deltas"],
                              "variant": st["variant"]}), flush=True)
            prob.close()


if __name__ == "__main__":
    main()
