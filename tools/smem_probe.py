"""Per-iteration cost of the shared-memory loops on tiny: iteration-kernel device time
(library events) for several run lengths, refresh cadences and lane counts."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PCDM_DEBUG_KNOBS", "1")

import torch  # noqa: E402

from paper_1212_0873_b200 import instances as I  # noqa: E402
from paper_1212_0873_b200 import pcdm  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    inst = I.generate("tiny", seed=0).to(dev)
    forms = [("0", "16"), ("1", "1"), ("1", "2"), ("1", "4"), ("1", "16")]
    iters_list = (20, 200, 2000, 8000)
    refreshes = (0, -1)
    if len(sys.argv) > 1:  # one form: smem1 lanes iters (ncu captures)
        forms = [(sys.argv[1], sys.argv[2])]
        iters_list = (int(sys.argv[3]),)
        refreshes = (0,)
    with pcdm.Problem.from_instance(inst) as prob:
        for smem1, lanes in forms:
            os.environ["PCDM_SMEM1"] = smem1
            os.environ["PCDM_SMEM_LANES"] = lanes
            for refresh in refreshes:
                for iters in iters_list:
                    best = None
                    for rep in range(5):
                        x = torch.zeros(inst.n, dtype=torch.float32, device=dev)
                        prob.run(x, 32, iters, seed=0, refresh_every=refresh, variant="smem")
                        st = prob.stats()
                        t = st["iter_kernel_ms"]
                        best = t if best is None else min(best, t)
                    print("smem1=%s lanes=%-2s refresh=%-2d iters=%-5d kernel_ms=%.4f us/iter=%.3f threads=%d nz=%d"
                          % (smem1, lanes, refresh, iters, best, 1e3 * best / iters, st["threads_per_cta"],
                             st["nonzero_deltas"]), flush=True)


if __name__ == "__main__":
    main()
