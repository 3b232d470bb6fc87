"""Multi-process host logic of the multi-GPU path on CPU (gloo, world_size 2).

The hot path shards (b, h) slices / batches across ranks with no exchange step
(SURVEY 8(e)); the only collectives are the barrier and the max-reduction of
per-rank timings.  These tests run that logic with the gloo backend and check
that every rank gets the max and that the job value follows weak scaling."""

import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    assert bench.dist_env() == (rank, world, rank)
    # per-rank step time: rank r is (r + 1) ms
    m = bench.reduce_max_ms(float(rank + 1), dist, "cpu")
    dist.barrier()
    # each rank generates its own shard of the synthetic batch (seed = rank): distinct data
    import hla_synth
    x = hla_synth.uniform_torch((1, 16, 1, 8), rank, 1)
    g = [torch.zeros_like(x.float()) for _ in range(world)]
    dist.all_gather(g, x.float())
    out[rank] = (m, bench.job_value(m, world), bool(torch.equal(g[0], g[1])))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_max_over_ranks_and_weak_scaling(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        m, v, same = res[r]
        assert m == float(world)                 # max over ranks
        assert v == float(world) / world         # ms per batch of work for the whole job
        assert not same                          # shards differ (seeded per rank)
