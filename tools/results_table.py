"""Markdown rows of BASELINE.md's "Measured results" table from bench.py JSON lines.

    python tools/results_table.py profiles/r02_configs.jsonl
"""
import json
import sys


def fmt(v, f="%.3g"):
    return "—" if v is None else (f % v)


def main(path):
    print("| Config | τ | loop | F rel (first step) | samples / ω exact | GPU updates/s | ms per step | "
          "roofline (bound, achieved/peak) | traffic (kind, frac) | oracle updates/s (1 core) |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        c = d["config"]
        par = d.get("parity") or {}
        rf = d["roofline"]
        cpu = d.get("cpu_baseline") or {}
        exact = "—" if not par else "%s / %s" % ("yes" if par.get("samples_bitexact") else "no",
                                                 "yes" if par.get("omega_bitexact") else "no")
        print("| %s | %s | %s | %s | %s | %s | %.2f | %s %.0f/%.0f GB/s = %.3f | %s | %s |" % (
            c["workload"], c["tau"], d.get("variant"), fmt(par.get("relF"), "%.1e"), exact, fmt(d["value"]),
            d["ms_per_step"], rf["bound"], rf["achieved"], rf["peak"], rf["frac"],
            "%s %.2f" % (rf["traffic_kind"], rf["traffic_frac"]) if rf.get("traffic_frac") else "—",
            fmt(cpu.get("value"))))


if __name__ == "__main__":
    main(sys.argv[1])
