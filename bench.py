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
VARIANT_NAMES = {1: "grid", 2: "smem", 3: "block", 4: "packed", 5: "batched", -1: "async"}
KERNEL_OF_VARIANT = {1: "pcdm_iter_kernel", 2: "pcdm_smem1_kernel", 3: "pcdm_iter_kernel",
                     4: "pcdm_packed_kernel (pcdm_packed1_kernel when the grid covers tau in one round, "
                        "pcdm_ragged_kernel on the ragged layout)",
                     5: "batch_expand+batch_sweep+screen_test (+screen_fix on its own stream, under the next expand)",
                     -1: "pcdm_async_kernel"}
# The oracle timing sample, per config (one definition for the cpu_baseline of our
# arm and for every step of --impl reference): iterations k = 0..K'-1 of the
# config's run from x_0 = 0, on the columns they touch, O5-O8 loop time only.
CPU_BASELINE_ITERS = {"tiny": 2000, "medium": 2000, "skewed": 200, "large": 60, "huge": 24, "logistic_small": 1000,
                      "kddb_like": 24, "ragged": 60, "ragged_small": 400}
L2_PEAK = (18571.5, "measured: profiles/r01_microbench.jsonl stream_read over a 66 MB buffer (L2-resident), "
                    "best of 100 reps")


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9
    except (ValueError, OSError):
        ram = None
    return {"host_cpu": model, "host_nproc": os.cpu_count(), "host_ram_gb": ram}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None,
                    choices=list(I.CONFIGS) + list(I.RAGGED_CONFIGS) + list(I.LOGISTIC_CONFIGS),
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
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the oracle parity check of the first step (samples, omega, F, x)")
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
    return I.generate(config_of(args), seed=0, device=device)


def config_of(args):
    if args.loss == "logistic":
        return I.LOGISTIC_CONFIGS[args.config]
    return I.CONFIGS[args.config] if args.config in I.CONFIGS else I.RAGGED_CONFIGS[args.config]


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
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""
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
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def ncu_traffic(config, variant, sampling, iters_per_launch, tau=None):
    """DRAM (and L2) bytes per iteration-kernel launch from the committed ncu capture of
    exactly this config, loop and sampling ("<config>:<loop>:<sampling>", written by
    tools/ncu_traffic.py), or None when that combination was not captured."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            table = json.load(f)
        # a capture of this tau first ("<config>@<tau>:..."), else the config's own
        d = table.get("%s@%s:%s:%s" % (config, tau, variant, sampling)) or table["%s:%s:%s" % (config, variant, sampling)]
    except Exception:
        return None
    out = {"dram": float(d["dram_bytes_per_iter"]) * iters_per_launch, "source": d.get("source"),
           "kernel": d.get("kernel")}
    if d.get("l2_bytes_per_iter") is not None:
        out["l2"] = float(d["l2_bytes_per_iter"]) * iters_per_launch
    return out


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


def oracle_slots(tau, k0, k_iters, seed, n, osamp=None):
    """The oracle's own slot arrays of S_k0..S_{k0+K-1} (int32[K, tau], -1 = idle)."""
    import oracle
    if osamp is None:
        return oracle.samples(seed, k0, k_iters, tau, n)
    return np.stack([oracle.sample_kind(osamp, seed, k, n) for k in range(k0, k0 + k_iters)])


def oracle_subinstance(inst, tau, k0, k_iters, seed, osamp=None, slots=None):
    """Host CSC holding only the columns S_k0..S_{k0+K-1} touch (others empty),
    gathered from the resident instance; the slots come from the oracle's own
    sampler.  Test/baseline infrastructure: never on the product path."""
    S = oracle_slots(tau, k0, k_iters, seed, inst.n, osamp) if slots is None else slots
    cols = np.unique(S)
    cols = cols[cols >= 0].astype(np.int64)
    c, r, v = I.column_subset(inst.colptr, inst.rowidx, inst.val, cols)
    return c, r, v, inst.b.cpu().numpy()


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


def cpu_sample_note(kcpu, cfg, tau, secs):
    return ("iterations k=0..%d of the %s run (tau=%d, seed 0, x_0 = 0) on the columns they touch; "
            "O5-O8 loop time %.2f s" % (kcpu - 1, cfg.name, tau, secs))


class ParityLeg:
    """Oracle parity of the bench's own first step (iterations 0..iters-1 from x_0 = 0,
    run seed 0): the oracle's slot arrays of every iteration, omega counted by the
    oracle over the whole matrix, and the oracle run of the same iterations on the
    columns they touch (alg:PCD1), forked into a background process
    so that it overlaps the GPU measurement.  Nothing it compares against comes from
    the CUDA path."""

    def __init__(self, inst, tau, iters, osamp):
        import tempfile

        import oracle
        from oracle.background import Job
        self.iters, self.tau, self.n, self.osamp = iters, tau, inst.n, osamp
        t0 = time.time()
        self.S = oracle_slots(tau, 0, iters, 0, inst.n, osamp)
        cols = np.unique(self.S)
        self.cols = cols[cols >= 0].astype(np.int64)
        colptr, rows, vals = I.column_subset(inst.colptr, inst.rowidx, inst.val, self.cols)
        b = inst.b.cpu().numpy()
        full_rows = inst.rowidx.cpu().numpy()
        m, lam = inst.m, inst.lam
        self.prep_s = time.time() - t0
        self.tmp = tempfile.mkdtemp(prefix="pcdm_bench_parity_")
        keep = self.cols

        def fn():
            om = oracle.omega(m, full_rows)  # O1 over the full matrix
            res = oracle.run(m, colptr, rows, vals, b, lam, tau, iters, 0, omega_override=om, sampling=osamp)
            F = oracle.objective(m, colptr, rows, vals, b, lam, res.x)
            return dict(x=res.x[keep], F=np.float64(F), omega=np.int64(om), beta=np.float64(res.beta),
                        loop_seconds=np.float64(res.loop_seconds))
        self.job = Job("parity", fn, self.tmp)

    def gpu_side(self, pcdm, prob, x, gsamp, dev):
        """Right after the first step: the GPU's slot arrays, F and x."""
        got = torch.empty(self.iters * self.tau, dtype=torch.int32, device=dev)
        if gsamp is None:
            pcdm.pcdm_sample(self.n, self.tau, 0, 0, self.iters, got)
        else:
            pcdm.pcdm_sample_sampling(self.n, gsamp, 0, 0, self.iters, got)
        self.samples_bitexact = bool(np.array_equal(got.cpu().numpy().reshape(self.S.shape), self.S))
        del got
        self.S = None
        self.F_gpu = prob.objective(x)
        xh = x.cpu().numpy()
        untouched = np.ones(xh.size, dtype=bool)
        untouched[self.cols] = False
        self.x_untouched_zero = not bool(np.any(xh[untouched]))
        self.x_gpu = xh[self.cols].astype(np.float64)

    def fields(self, omega_gpu):
        import shutil
        res = self.job.result()
        shutil.rmtree(self.tmp, ignore_errors=True)
        F_o = float(res["F"])
        xo = res["x"]
        scale = max(float(np.max(np.abs(xo))) if xo.size else 0.0, 1e-30)
        dx = float(np.max(np.abs(self.x_gpu - xo))) / scale if xo.size else 0.0
        relF = abs(self.F_gpu - F_o) / abs(F_o)
        omega_ok = int(res["omega"]) == int(omega_gpu)
        green = self.samples_bitexact and omega_ok and relF <= 1e-5 and dx <= 1e-4 and self.x_untouched_zero
        return {"scope": "first step: iterations 0..%d from x_0 = 0, seed 0; oracle on the %d columns they touch, "
                         "omega over the full matrix" % (self.iters - 1, self.cols.size),
                "samples_bitexact": self.samples_bitexact, "omega_bitexact": omega_ok,
                "omega_oracle": int(res["omega"]), "F_gpu": self.F_gpu, "F_oracle": F_o, "relF": relF,
                "dx_rel": dx, "x_untouched_zero": self.x_untouched_zero,
                "tolerance": {"relF": 1e-5, "dx_rel": 1e-4}, "status": "green" if green else "FAIL",
                "oracle_loop_s": float(res["loop_seconds"]), "oracle_wall_s": float(res["wall_s"]),
                "prep_s": self.prep_s}


# ----------------------------------------------------------------------------- arms
def bench_reference(args, world, rank):
    if rank != 0:
        return
    cfg = config_of(args)
    tau = args.tau or cfg.tau
    kcpu = CPU_BASELINE_ITERS[args.config]
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    inst = make_instance(args, dev)
    avg_c = inst.nnz / inst.n
    K, W = args.steps, args.warmup
    osamp = oracle_sampling(args, tau)
    sub = oracle_subinstance(inst, tau, 0, kcpu, seed=0, osamp=osamp)
    del inst.rowidx, inst.val
    secs = []
    for s in range(W + K):
        t, _ = run_oracle_sample(inst, tau, 0, kcpu, 0, sub=sub, osamp=osamp, loss=args.loss)
        if s >= W:
            secs.append(t)
    step_s = sum(secs) / len(secs)
    value = expected_size(args.sampling, tau, inst.n, args.p_b) * kcpu / step_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": 1,
            "steps": K, "warmup": W, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "nnz_per_col": cfg.nnz_per_col,
                       "tau": tau, "sampling": args.sampling, "iters_per_step": kcpu, "seed": 0,
                       "note": "serial oracle on one host core; every step is the same bounded sample as our "
                               "arm's cpu_baseline"},
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": 1, "kind": "oracle",
                             "sample": cpu_sample_note(kcpu, cfg, tau, step_s)},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "effective_GBps": value * avg_c * BYTES_PER_NNZ / 1e9}
    line.update(host_info())
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
    gsamp = None if args.sampling == "nice" else pcdm.Sampling(args.sampling, tau, p_b=args.p_b)
    osamp = oracle_sampling(args, tau) if rank == 0 and world == 1 else None
    # oracle parity of the first step (run seed 0 = rank 0), started before create so the
    # host copies are taken while device memory is free; it runs in the background
    parity = None
    do_parity = (rank == 0 and world == 1 and not args.no_parity and args.loss == "lasso" and not args.async_)
    if do_parity:
        parity = ParityLeg(inst, tau, iters, osamp)
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
    if do_cpu:
        sub = oracle_subinstance(inst, tau, 0, kcpu, seed=0, osamp=osamp)
    del inst.rowidx, inst.val
    torch.cuda.empty_cache()

    run_seed = rank
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

    for w in range(W):
        one_step(x)
        if w == 0 and parity is not None:
            torch.cuda.synchronize()
            parity.gpu_side(pcdm, prob, x, gsamp, dev)
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
    # bound: HBM when r (gathered and scattered every iteration) does not fit in L2,
    # else the L2 (A streams from HBM or sits in L2, r is served by L2)
    r_in_l2 = 4 * inst.m <= l2_bytes // 2
    hpeak, hpeak_src = hbm_peak()
    peak, peak_src = (L2_PEAK if r_in_l2 else (hpeak, hpeak_src))
    samp_key = args.sampling if args.sampling != "binomial" else "binomial%g" % args.p_b
    traffic = None if args.async_ else ncu_traffic(cfg.name, VARIANT_NAMES.get(st_list[-1]["variant"], "?"),
                                                    samp_key, iters_per_launch, tau)
    # ncu traffic of the bounding memory level: DRAM bytes for HBM-bound runs, L2 bytes
    # (lts__t_bytes) for L2-bound ones
    traffic_kind = ("l2" if r_in_l2 else "dram") if traffic else None
    traffic_bytes = traffic.get(traffic_kind) if traffic else None
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
        if parity is not None:
            parity.job.result()  # the timing sample runs alone on the host
        secs, _ = run_oracle_sample(inst, tau, 0, kcpu, 0, sub=sub, osamp=osamp, loss=args.loss)
        cpu = {"value": size * kcpu / secs, "unit": "updates/s", "cores": 1, "kind": "oracle",
               "sample": cpu_sample_note(kcpu, cfg, tau, secs)}
    par = parity.fields(prob.omega) if parity is not None else None

    if rank != 0:
        return
    st0 = st_list[-1]
    line = {
        "metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "nnz": nnz, "nnz_per_col": cfg.nnz_per_col
                   if cfg.col_lengths == "fixed" else "pareto(alpha=%g, %d..%d), mean %.2f"
                   % (cfg.len_alpha, cfg.len_min, cfg.len_max, avg_c),
                   "rows": cfg.rows, "tau": tau, "iters_per_step": iters, "seed_instance": 0, "loss": args.loss,
                   "sampling": args.sampling if args.sampling != "binomial" else "binomial(p_b=%g)" % args.p_b,
                   "seed_run": "rank", "parallelism": "replicas" if world > 1 else "single",
                   "l2": ("inputs larger than L2 (A %.1f GB vs L2 %.0f MB)" % (nnz * 8 / 1e9, l2_bytes / 1e6))
                   if flush is None else "L2 flushed between timed steps"},
        "effective_GBps": value * avg_c * BYTES_PER_NNZ / 1e9,
        "roofline": {"bound": "l2" if r_in_l2 else "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic_bytes, "peak_source": peak_src,
                     "traffic_kind": traffic_kind, "traffic_source": traffic["source"] if traffic else None,
                     "traffic_GBps": traffic_bytes / (launch_ms / 1e3) / 1e9 if traffic_bytes else None,
                     "traffic_frac": traffic_bytes / (launch_ms / 1e3) / 1e9 / peak if traffic_bytes else None,
                     "dram_traffic_frac_of_hbm": traffic["dram"] / (launch_ms / 1e3) / 1e9 / hpeak
                     if traffic else None,
                     "hbm_peak": hpeak,
                     "kernel": (traffic or {}).get("kernel") or KERNEL_OF_VARIANT.get(st0["variant"], "?"),
                     "algorithmic_bytes_per_launch": alg_bytes_launch,
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
        "screen_per_step": {f: sum(s.get("screen_" + f, 0) for s in st_list) / K
                            for f in ("misses", "scans", "spec", "flagged")},
        "grid": {"ctas": st0["grid_ctas"], "threads": st0["threads_per_cta"], "lanes_per_column": st0["lanes_per_column"]},
        "setup_s": {"generate": gen_s, "create": create_s},
        "parity": par,
        "context": "paper: 2e10-nnz LASSO in ~2 h on 24 cores (~4.8e6 updates/s, asynchronous, PAPER.md:1237,1248)",
    }
    line.update(host_info())
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
