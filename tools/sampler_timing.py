"""Device time of the tau-nice sampler alone (pcdm_sample: the same sample_chunk
passes pcdm_run uses, plus one device-to-device copy of the slots per chunk) for
the BASELINE configs' (n, tau), CUDA events on the launching stream."""
import json
import sys

import torch

from paper_1212_0873_b200 import pcdm

SHAPES = {"huge": (500_000_000, 1 << 18, 90), "large": (10_000_000, 65536, 200), "skewed": (1_000_000, 65536, 310)}


def main(names):
    dev = torch.device("cuda:0")
    for name in names:
        n, tau, count = SHAPES[name]
        out = torch.empty(count * tau, dtype=torch.int32, device=dev)
        st = torch.cuda.current_stream()
        for _ in range(2):
            pcdm.pcdm_sample(n, tau, 0, 0, count, out)
        ts = []
        for rep in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            pcdm.pcdm_sample(n, tau, 0, 1000 * rep, count, out)
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        print(json.dumps({"shape": name, "n": n, "tau": tau, "iters": count, "ms_median": ts[2],
                          "us_per_iter": 1e3 * ts[2] / count}), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SHAPES))
