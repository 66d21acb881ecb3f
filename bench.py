#!/usr/bin/env python
"""Benchmark of the PCDM1/LASSO hot path on B200 (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config huge|large|skewed|medium|tiny] [--tau T] [--iters I]

A "step" is one pcdm_run call of `iters` synchronous PCDM1 iterations (sampling,
gathers a_i^T r, soft-threshold steps, residual scatter, barriers) on the
config's synthetic instance; consecutive steps continue the same solve
(first_iter advances), so every step is real work on resident HBM inputs.
Metric: coordinate updates/s (= E|S| * iters per step; E|S| = tau for tau-nice), plus effective GB/s at
16 B per touched nonzero (val + idx + r gather + r scatter).

Multi-GPU (torchrun): replicas only -- every rank solves its own
replica with its own run seed; value = all ranks' updates / max-over-ranks time.

--impl reference times the oracle (oracle/, serial C, fp64) on host cores on a
bounded sample of the same workload (the first iterations of the same run on
the columns they touch); only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1212_0873_b200 import instances as I  # noqa: E402

METRIC = "coordinate updates/sec and effective GB/s (fraction of HBM/L2 roofline) at 1 B200"
BYTES_PER_NNZ = 16  # val 4 + idx 4 + r gather 4 + r scatter 4
VARIANT_NAMES = {1: "grid", 2: "smem", 3: "block", 4: "packed", 5: "batched", 6: "cluster", -1: "async"}
KERNEL_OF_VARIANT = {1: "pcdm_iter_kernel", 2: "pcdm_smem_kernel", 3: "pcdm_iter_kernel", 4: "pcdm_packed_kernel",
                     5: "batch_expand+batch_sweep+pcdm_batched_slot+batch_fold", 6: "pcdm_cluster_kernel",
                     -1: "pcdm_async_kernel"}
# oracle iterations per reference step / cpu_baseline sample, per config
REF_ITERS = {"tiny": 400, "medium": 200, "skewed": 20, "large": 8, "huge": 4, "logistic_small": 200, "kddb_like": 4}
CPU_BASELINE_ITERS = {"tiny": 2000, "medium": 2000, "skewed": 200, "large": 60, "huge": 24, "logistic_small": 1000,
                      "kddb_like": 24}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=list(I.CONFIGS) + list(I.LOGISTIC_CONFIGS),
                    help="default: huge (LASSO) / kddb_like (logistic)")
    ap.add_argument("--loss", default="lasso", choices=["lasso", "logistic"],
                    help="logistic: the L2-regularised logistic problem of Sec. 8.4 (NEXT-3)")
    ap.add_argument("--tau", type=int, default=None)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--sampling", default="nice", choices=["nice", "independent", "binomial"],
                    help="doubly uniform sampling (NEXT-1 rows); the headline is tau-nice")
    ap.add_argument("--p-b", type=float, default=0.5, help="binomial availability probability")
    ap.add_argument("--async", dest="async_", action="store_true",
                    help="asynchronous variant (NEXT-4, PAPER.md:1248): tau*iters updates per step, no barriers")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    a = ap.parse_args()
    if a.config is None:
        a.config = "kddb_like" if a.loss == "logistic" else "huge"
    return a


class LogisticInstance:
    """The synthetic KDDB-shaped logistic instance in the shape bench.py uses (b = labels y)."""

    def __init__(self, cfg, device):
        self.cfg = I.LOGISTIC_CONFIGS[cfg] if isinstance(cfg, str) else cfg
        self.colptr, self.rowidx, self.val, self.b, self.lam = I.generate_logistic(self.cfg, seed=0, device=device)
        self.m, self.n = self.cfg.m, self.cfg.n

    @property
    def nnz(self):
        return int(self.rowidx.numel())


def make_instance(args, device):
    if args.loss == "logistic":
        return LogisticInstance(args.config, device)
    return I.generate(I.CONFIGS[args.config], seed=0, device=device)


def config_of(args):
    return I.LOGISTIC_CONFIGS[args.config] if args.loss == "logistic" else I.CONFIGS[args.config]


# ----------------------------------------------------------------------------- dist
def dist_setup(args=None):
    """One process per GPU (torchrun env).  NCCL when CUDA is present, gloo on a
    CPU-only host (the multi-process path is tested there with world_size 2)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(v, world):
    """Max over ranks (the slowest rank's step time defines the job's time)."""
    if world == 1:
        return v
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank_step, rank_ms_per_step, world):
    """Whole-job value: units all ranks processed per step / max-over-ranks step time (weak scaling:
    every rank solves its own replica).  Returns (value, ms_per_step)."""
    ms = allreduce_max(rank_ms_per_step, world)
    return units_per_rank_step * world / (ms / 1e3), ms


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.05)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.th.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- peaks
def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(config, variant, iters_per_launch):
    """DRAM bytes per iteration-kernel launch from the committed ncu capture of this
    config and loop ("<config>:<variant>"), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)["%s:%s" % (config, variant)]
        return float(d["dram_bytes_per_iter"]) * iters_per_launch
    except Exception:
        return None


# ----------------------------------------------------------------------------- oracle sample
def expected_size(kind, tau, n, p_b):
    """E|S| of the sampling (tau-nice: tau; binomial: tau p_b; tau-independent:
    occupied bins of tau balls in n bins) -- used only to count coordinate updates."""
    if kind == "binomial":
        return tau * p_b
    if kind == "independent":
        return -n * np.expm1(tau * np.log1p(-1.0 / n))
    return float(tau)


def oracle_sampling(args, tau):
    import oracle
    return None if args.sampling == "nice" else oracle.Sampling(args.sampling, tau, p_b=args.p_b)


def oracle_subinstance(inst, tau, k0, k_iters, seed, osamp=None):
    """Host CSC holding only the columns S_k0..S_{k0+K-1} touch (others empty),
    gathered from the resident instance; the slots come from the oracle's own
    sampler.  Test/baseline infrastructure: never on the product path."""
    import oracle
    n = inst.n
    S = [oracle.sample(seed, k, tau, n) if osamp is None else oracle.sample_kind(osamp, seed, k, n)
         for k in range(k0, k0 + k_iters)]
    cols = np.unique(np.concatenate(S)).astype(np.int64)
    cols = cols[cols >= 0]
    dev = inst.colptr.device
    ct = torch.from_numpy(cols).to(dev)
    starts = inst.colptr[ct]
    lens = inst.colptr[ct + 1] - starts
    total = int(lens.sum())
    offs = torch.cumsum(lens, 0) - lens
    idx = torch.repeat_interleave(starts - offs, lens) + torch.arange(total, device=dev)
    rows = inst.rowidx[idx].cpu().numpy()
    vals = inst.val[idx].cpu().numpy()
    full = np.zeros(n + 1, dtype=np.int64)
    full[cols + 1] = lens.cpu().numpy()
    np.cumsum(full, out=full)
    return full, rows, vals, inst.b.cpu().numpy()


def run_oracle_sample(inst, tau, k0, k_iters, seed, sub=None, osamp=None, loss="lasso"):
    import oracle
    if sub is None:
        sub = oracle_subinstance(inst, tau, k0, k_iters, seed, osamp)
    c, r, v, b = sub
    if loss == "logistic":
        res = oracle.logistic_run(inst.m, c, r, v, b, inst.lam, tau, k_iters, seed, first_iter=k0, sampling=osamp)
    else:
        res = oracle.run(inst.m, c, r, v, b, inst.lam, tau, k_iters, seed, first_iter=k0, sampling=osamp)
    return res.loop_seconds, sub


# ----------------------------------------------------------------------------- arms
def bench_reference(args, world, rank):
    if rank != 0:
        return
    cfg = config_of(args)
    tau = args.tau or cfg.tau
    kref = REF_ITERS[args.config]
    dev = torch.device("cuda", 0)
    inst = make_instance(args, dev)
    K, W = args.steps, args.warmup
    osamp = oracle_sampling(args, tau)
    sub = oracle_subinstance(inst, tau, 0, kref * (K + W), seed=0, osamp=osamp)
    del inst.rowidx, inst.val
    secs = []
    for s in range(W + K):
        t, _ = run_oracle_sample(inst, tau, s * kref, kref, 0, sub=sub, osamp=osamp, loss=args.loss)
        if s >= W:
            secs.append(t)
    step_s = sum(secs) / len(secs)
    value = expected_size(args.sampling, tau, inst.n, args.p_b) * kref / step_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": 1,
            "steps": K, "warmup": W, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "nnz_per_col": cfg.nnz_per_col,
                       "tau": tau, "sampling": args.sampling, "iters_per_step": kref, "seed": 0,
                       "note": "serial oracle on host cores; each step = %d iterations of the same run" % kref},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": 1, "kind": "oracle",
                             "sample": "iterations k=%d..%d of the %s run (columns they touch), O5-O8 loop only"
                                       % (W * kref, (W + K) * kref - 1, cfg.name)},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "effective_GBps": value * cfg.nnz_per_col * BYTES_PER_NNZ / 1e9}
    print(json.dumps(line), flush=True)


def bench_ours(args, world, rank, local):
    from paper_1212_0873_b200 import build as pbuild
    from paper_1212_0873_b200 import pcdm
    if rank == 0:
        pbuild.build()
    barrier(world)
    pcdm.load()
    cfg = config_of(args)
    tau = args.tau or cfg.tau
    iters = args.iters or cfg.iters
    K, W = args.steps, args.warmup
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    t0 = time.time()
    inst = make_instance(args, dev)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    t0 = time.time()
    prob = pcdm.Problem(inst.m, inst.n, inst.colptr, inst.rowidx, inst.val, inst.b, inst.lam, loss=args.loss)
    create_s = time.time() - t0
    nnz = inst.nnz
    avg_c = nnz / inst.n
    working_set = inst.nnz * 8 + inst.m * 4
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size

    # bounded oracle sample for the cpu_baseline, built while A is still ours to read
    sub = None
    do_cpu = (rank == 0 and world == 1 and not args.no_cpu_baseline)
    kcpu = CPU_BASELINE_ITERS[args.config]
    osamp = oracle_sampling(args, tau) if do_cpu else None
    if do_cpu:
        sub = oracle_subinstance(inst, tau, 0, kcpu, seed=0, osamp=osamp)
    del inst.rowidx, inst.val
    torch.cuda.empty_cache()

    run_seed = rank
    gsamp = None if args.sampling == "nice" else pcdm.Sampling(args.sampling, tau, p_b=args.p_b)
    size = expected_size(args.sampling, tau, inst.n, args.p_b)
    x = torch.zeros(inst.n, dtype=torch.float32, device=dev)
    flush = torch.empty(int(2 * l2_bytes) // 4, dtype=torch.float32, device=dev) \
        if working_set < 4 * l2_bytes else None
    step = 0

    def one_step(xbuf):
        nonlocal step
        if args.async_:
            prob.run_async(xbuf, tau * iters, seed=run_seed, first_update=step * tau * iters, stream=stream)
            step += 1
            return
        prob.run(xbuf, tau, iters, seed=run_seed, first_iter=step * iters, variant=args.variant, sampling=gsamp,
                 stream=stream)
        step += 1

    for _ in range(W):
        one_step(x)
    torch.cuda.synchronize()
    barrier(world)
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    st_list = []
    for s in range(K):
        if flush is not None:
            flush.fill_(float(s))
        ev[s][0].record(stream)
        one_step(x)
        ev[s][1].record(stream)
        st_list.append(prob.stats())
    torch.cuda.synchronize()
    barrier(world)
    clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    updates_per_step = size * iters
    value, ms_per_step = job_throughput(updates_per_step, sum(step_ms) / K, world)
    F_final = prob.objective(x)

    # roofline of the dominant kernel (the persistent iteration kernel)
    it_ms = sum(s["iter_kernel_ms"] for s in st_list)
    it_launches = sum(s["iter_launches"] for s in st_list)
    samp_ms = sum(s["sampler_ms"] for s in st_list)
    setup_ms = sum(s["setup_ms"] for s in st_list)
    iters_per_launch = K * iters / max(it_launches, 1)  # async: tau updates count as one "iteration"
    alg_bytes_launch = BYTES_PER_NNZ * avg_c * size * iters_per_launch
    launch_ms = it_ms / max(it_launches, 1)
    achieved = alg_bytes_launch / (launch_ms / 1e3) / 1e9
    peak, peak_src = hbm_peak()
    traffic = None if args.async_ else ncu_traffic(cfg.name, VARIANT_NAMES.get(st_list[-1]["variant"], "?"),
                                                    iters_per_launch)
    launches = sum(s["kernel_launches"] for s in st_list)
    nz = sum(s["nonzero_deltas"] for s in st_list)

    # end-to-end through the C ABI with a pinned HOST x: H2D + run + D2H per step
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        ke = max(1, min(K, 3))
        eve = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ke)]
        one_step(xh)  # untimed: the host-x path's one-time allocations (staging, side stream)
        torch.cuda.synchronize()
        h2d = d2h = 0
        for s in range(ke):
            eve[s][0].record(stream)
            one_step(xh)
            eve[s][1].record(stream)
            st_e = prob.stats()
            h2d += st_e.get("host_h2d_bytes", inst.n * 4)
            d2h += st_e.get("host_d2h_bytes", inst.n * 4)
        torch.cuda.synchronize()
        e2e_value, e2e_ms = job_throughput(updates_per_step, sum(a.elapsed_time(b) for a, b in eve) / ke, world)
        e2e = {"value": e2e_value, "unit": "updates/s",
               "h2d_bytes_per_step": h2d // ke, "d2h_bytes_per_step": d2h // ke,
               "ms_per_step": e2e_ms, "steps": ke,
               "note": "pcdm_run_ex on pinned host x: x H2D, run, changed entries of x D2H (the library's "
                       "compact copy-back, host_d2h_bytes) inside the timed region"}

    cpu = None
    if do_cpu:
        secs, _ = run_oracle_sample(inst, tau, 0, kcpu, 0, sub=sub, osamp=osamp, loss=args.loss)
        cpu = {"value": size * kcpu / secs, "unit": "updates/s", "cores": 1, "kind": "oracle",
               "sample": "iterations k=0..%d of the %s run (tau=%d) on the columns they touch; "
                         "O5-O8 loop time %.2f s" % (kcpu - 1, cfg.name, tau, secs)}

    if rank != 0:
        return
    st0 = st_list[-1]
    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "nnz": nnz, "nnz_per_col": cfg.nnz_per_col,
                   "rows": cfg.rows, "tau": tau, "iters_per_step": iters, "seed_instance": 0, "loss": args.loss,
                   "sampling": args.sampling if args.sampling != "binomial" else "binomial(p_b=%g)" % args.p_b,
                   "seed_run": "rank", "parallelism": "replicas" if world > 1 else "single",
                   "l2": ("inputs larger than L2 (A %.1f GB vs L2 %.0f MB)" % (nnz * 8 / 1e9, l2_bytes / 1e6))
                   if flush is None else "L2 flushed between timed steps"},
        "effective_GBps": value * avg_c * BYTES_PER_NNZ / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "traffic_GBps": traffic / (launch_ms / 1e3) / 1e9 if traffic else None,
                     "traffic_frac": traffic / (launch_ms / 1e3) / 1e9 / peak if traffic else None,
                     "kernel": KERNEL_OF_VARIANT.get(st0["variant"], "?"), "algorithmic_bytes_per_launch": alg_bytes_launch,
                     "launch_ms": launch_ms, "iters_per_launch": iters_per_launch,
                     "share_of_step": it_ms / max(sum(step_ms), 1e-9)},
        "breakdown_ms_per_step": {"iteration_kernel": it_ms / K, "sampler": samp_ms / K, "setup": setup_ms / K},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "omega": prob.omega, "beta": prob.beta(tau) if gsamp is None else prob.beta_sampling(gsamp),
        "async": bool(args.async_),
        "F_final": F_final, "nonzero_step_frac": nz / (K * size * iters),
        "variant": VARIANT_NAMES.get(st0["variant"], "?"),
        "grid": {"ctas": st0["grid_ctas"], "threads": st0["threads_per_cta"], "lanes_per_column": st0["lanes_per_column"]},
        "setup_s": {"generate": gen_s, "create": create_s},
        "context": "paper: 2e10-nnz LASSO in ~2 h on 24 cores (~4.8e6 updates/s, asynchronous, PAPER.md:1237,1248)",
    }
    print(json.dumps(line), flush=True)
    prob.close()


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            bench_reference(args, world, rank)
        else:
            bench_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
