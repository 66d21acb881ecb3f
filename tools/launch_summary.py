"""Summarise an `ncu --csv --log-file` metrics capture: per kernel, mean duration,
DRAM bytes read/written per launch and the achieved DRAM rate."""
import collections
import csv
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(lines[start:]))


def summary(path):
    agg = collections.OrderedDict()
    for r in load(path):
        k = r["Kernel Name"].split("(")[0].replace("void <unnamed>::", "").replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if unit in ("nsecond", "ns"):
            v /= 1e3
        elif unit in ("msecond", "ms"):
            v *= 1e3
        if unit in ("Kbyte",):
            v *= 1e3
        if unit in ("Mbyte", "MB"):
            v *= 1e6
        if unit in ("Gbyte", "GB"):
            v *= 1e9
        agg.setdefault(k, collections.defaultdict(list))[r["Metric Name"]].append(v)
    out = []
    for k, m in agg.items():
        t = m.get("gpu__time_duration.sum", [0])
        n = len(t)
        us = sum(t) / n
        rd = sum(m.get("dram__bytes_read.sum", [0])) / n
        wr = sum(m.get("dram__bytes_write.sum", [0])) / n
        out.append((k, n, us, rd, wr, (rd + wr) / (us * 1e-6) / 1e12 if us else 0.0))
    return out


if __name__ == "__main__":
    for k, n, us, rd, wr, tbs in summary(sys.argv[1]):
        print("%-40s n=%-4d %9.1f us  read %8.1f MB  write %8.1f MB  %.2f TB/s" % (k[:40], n, us, rd / 1e6, wr / 1e6, tbs))
