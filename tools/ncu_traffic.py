"""Record the DRAM (and L2) traffic per iteration of one (config, loop, sampling) from an
ncu metrics capture, for bench.py's roofline.traffic (profiles/ncu_traffic.json).

    python tools/ncu_traffic.py CAPTURE.csv KEY ITERS_PER_LAUNCH [--kernels REGEX] [--note TEXT]

CAPTURE.csv: `ncu --csv --log-file` output with dram__bytes_read.sum,
dram__bytes_write.sum (and optionally lts__t_bytes.sum) per kernel launch.  The kernels
matching REGEX that make up one iteration-kernel launch (e.g. one chunk of the batched
loop: expand, sweep, test, fix) are averaged per launch and summed; the result divided by
ITERS_PER_LAUNCH is stored under KEY = "<config>:<loop>:<sampling>".
"""
import argparse
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from launch_summary import load  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def per_launch(path, regex, total=False):
    acc = {}
    for r in load(path):
        name = r["Kernel Name"]
        if not re.search(regex, name):
            continue
        k = name.split("(")[0]
        v = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
        acc.setdefault(k, {}).setdefault(r["Metric Name"], []).append(v)
    out = {"dram": 0.0, "l2": 0.0, "kernels": {}}
    for k, m in acc.items():
        rd = m.get("dram__bytes_read.sum", [0.0])
        wr = m.get("dram__bytes_write.sum", [0.0])
        l2 = m.get("lts__t_bytes.sum")
        div = 1 if total else len(rd)
        d = (sum(rd) + sum(wr)) / div
        out["dram"] += d
        out["kernels"][k] = {"dram_bytes": d, "launches": len(rd)}
        if l2:
            out["l2"] += sum(l2) / (1 if total else len(l2))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("capture")
    ap.add_argument("key")
    ap.add_argument("iters_per_launch", type=float)
    ap.add_argument("--kernels", default=".")
    ap.add_argument("--note", default="")
    ap.add_argument("--total-iters", type=float, default=None,
                    help="the capture holds every launch of runs totalling this many iterations: "
                         "bytes summed over the launches (ITERS_PER_LAUNCH then ignored)")
    a = ap.parse_args()
    t = per_launch(a.capture, a.kernels, total=a.total_iters is not None)
    if a.total_iters is not None:
        a.iters_per_launch = a.total_iters
    d = json.load(open(OUT)) if os.path.exists(OUT) else {}
    d[a.key] = {"dram_bytes_per_iter": t["dram"] / a.iters_per_launch,
                "l2_bytes_per_iter": (t["l2"] / a.iters_per_launch) if t["l2"] else None,
                "source": "%s (%s)%s" % (os.path.relpath(a.capture, ROOT), ", ".join(
                    "%s %.1f MB" % (k.replace("void ", ""), v["dram_bytes"] / 1e6) for k, v in t["kernels"].items()),
                    ("; " + a.note) if a.note else ""),
                "kernel": "+".join(k.replace("void ", "").replace("<unnamed>::", "") for k in t["kernels"])}
    json.dump(d, open(OUT, "w"), indent=1)
    print(a.key, d[a.key])


if __name__ == "__main__":
    main()
