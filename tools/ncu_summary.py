#!/usr/bin/env python
"""Summarise ncu outputs into the compact files committed under profiles/.

    python tools/ncu_summary.py launches <launches.csv> [--only-lib]     per-kernel count / total / mean / share
    python tools/ncu_summary.py full <report.ncu-rep> [metric-substrings...]  selected raw metrics per launch

`launches` reads the CSV written by `ncu --metrics gpu__time_duration.sum --csv
--log-file ...`; with --only-lib the share is computed over libpcdm's kernels
only (torch kernels of the instance generator are dropped).
"""
import collections
import csv
import subprocess
import sys

LIB_KERNELS = ("pcdm_", "sample_", "neg_b_kernel", "scatter_x_kernel", "round_r_kernel", "validate_kernel",
               "check_finite_kernel", "row_counts_kernel", "max_kernel", "col_norms_kernel", "objective_sums_kernel",
               "pack_kernel", "max_len_kernel", "plan_", "batch_", "tile_")

DEFAULT_METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                   "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
                   "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_read.sum",
                   "l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                   "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
                   "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]


def short(name):
    base = name.split("(")[0]
    return base.replace("void ", "").replace("<unnamed>::", "").strip()


def to_ns(v, unit):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)


def launches(path, only_lib):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        nm = short(d["Kernel Name"])
        if only_lib and not any(k in nm for k in LIB_KERNELS):
            continue
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += to_ns(d["Metric Value"], d["Metric Unit"])
    tot = sum(v[1] for v in agg.values()) or 1.0
    print("kernel,launches,total_us,mean_us,share")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("%s,%d,%.1f,%.2f,%.4f" % (k, v[0], v[1] / 1e3, v[1] / 1e3 / v[0], v[1] / tot))


def full(path, metrics):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    print("kernel,metric,unit,value")
    for r in rows[2:]:
        for m in metrics:
            if m in h:
                i = h.index(m)
                print("%s,%s,%s,%s" % (short(r[ki]), m, units[i], r[i]))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], "--only-lib" in sys.argv)
    else:
        full(sys.argv[2], sys.argv[3:] or DEFAULT_METRICS)
