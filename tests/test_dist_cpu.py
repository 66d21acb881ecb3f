"""Multi-process path of bench.py on CPU (gloo, world_size 2).

The hot path does not shard at N <= 5 configs (replicas
only): each rank solves its own replica with run seed = rank, and the job's
value is all ranks' updates / the max-over-ranks step time.  These tests drive
bench.py's own rendezvous / barrier / max-reduction / aggregation helpers in two
real processes over gloo (127.0.0.1), and check that the replicas' sampling
streams are distinct (the oracle's sampler, test infrastructure).
"""
import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist

    import oracle
    w, r, local = bench.dist_setup()
    assert (w, r, local) == (world, rank, rank)
    assert dist.get_backend() == "gloo"
    bench.barrier(w)
    # rank 1 is the slow one: the job time is ITS step time
    ms = 10.0 if rank == 0 else 40.0
    value, ms_job = bench.job_throughput(1000, ms, w)
    # replica streams: run seed = rank
    s0 = oracle.sample(rank, 0, 8, 1000).tolist()
    gathered = [None] * w
    dist.all_gather_object(gathered, s0)
    with open(os.path.join(out_dir, "rank%d.json" % rank), "w") as f:
        json.dump({"value": value, "ms": ms_job, "samples": gathered}, f)
    dist.destroy_process_group()


def test_replicas_over_gloo_world2(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = [json.load(open(tmp_path / ("rank%d.json" % r))) for r in range(world)]
    for d in res:
        assert d["ms"] == pytest.approx(40.0)                       # max over ranks
        assert d["value"] == pytest.approx(2 * 1000 / 0.040)        # all ranks' units / max time
        assert d["samples"][0] != d["samples"][1]                   # distinct replica streams
        assert len(set(d["samples"][0])) == 8
    assert res[0]["samples"] == res[1]["samples"]


def test_single_process_helpers():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.allreduce_max(3.5, 1) == 3.5
    v, ms = bench.job_throughput(500, 20.0, 1)
    assert ms == 20.0 and v == pytest.approx(500 / 0.020)
