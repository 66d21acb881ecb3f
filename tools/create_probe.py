"""pcdm_create on a config, bracketed by cudaProfilerStart/Stop (ncu --profile-from-start
off captures the create kernels only); prints the wall time of create (best of N)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1212_0873_b200 import instances as I  # noqa: E402
from paper_1212_0873_b200 import pcdm  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "huge"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda:0")
    inst = I.generate(cfg, seed=0, device=dev)
    torch.cuda.synchronize()
    for rep in range(reps):
        if rep == reps - 1:
            torch.cuda.profiler.start()
        t0 = time.time()
        prob = pcdm.Problem.from_instance(inst)
        torch.cuda.synchronize()
        dt = time.time() - t0
        if rep == reps - 1:
            torch.cuda.profiler.stop()
        print("create %s rep %d: %.1f ms" % (cfg, rep, 1e3 * dt), flush=True)
        prob.close()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
