"""Host logic of the multi-GPU path on CPU (SURVEY 4.2 tier T4, 8(e)).

The hot path shards the B x H independent (batch, head) attention units over the ranks
with no exchange step; NCCL carries only the barrier, the max-reduction of step times and
the after-loop all_gather of per-rank statistics.  Here: the shard planner as a pure
function (every unit exactly once, contiguous blocks), and the world_size-2 run of the
planner + input shards + max + gather with the gloo backend."""

import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("B,H", [(16, 8), (16, 12), (128, 3), (128, 24), (1, 8), (2, 12), (4, 2), (1, 1), (3, 5)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plan_shards_covers_every_unit_once(B, H, world):
    plan = bench.plan_shards(B, H, world)
    if plan is None:
        # no batch x head partition: neither B nor a head split of one batch divides evenly
        assert B % world and (world % B or H % (world // B))
        return
    assert len(plan) == world
    owner = {}
    for r, (b0, b1, h0, h1) in enumerate(plan):
        assert 0 <= b0 < b1 <= B and 0 <= h0 < h1 <= H            # a non-empty contiguous block
        for b in range(b0, b1):
            for h in range(h0, h1):
                assert (b, h) not in owner
                owner[(b, h)] = r
    assert len(owner) == B * H                                       # every unit exactly once
    sizes = {(b1 - b0) * (h1 - h0) for b0, b1, h0, h1 in plan}
    assert sizes == {B * H // world}                                 # balanced (strong scaling)
    if B % world == 0:                                               # whole batches: contiguous memory
        assert all(h0 == 0 and h1 == H for _, _, h0, h1 in plan)


def test_cfg_partitions_match_north_star():
    # north_star / SURVEY 8(e): batch 16 -> 2 batches per rank at 8 GPUs (cfg2-4); cfg5 128 -> 16
    assert bench.plan_shards(16, 12, 8)[3] == (6, 8, 0, 12)
    assert bench.plan_shards(128, 3, 8)[7] == (112, 128, 0, 3)
    assert bench.plan_shards(1, 8, 4) == [(0, 1, 0, 2), (0, 1, 2, 4), (0, 1, 4, 6), (0, 1, 6, 8)]
    assert bench.plan_shards(1, 1, 2) is None                       # cfg1: replicas only


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
    import bench as bch
    import hla_synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    assert bch.dist_env() == (rank, world, rank)
    B, N, H, d = 4, 16, 3, 8
    b0, b1, h0, h1 = bch.plan_shards(B, H, world)[rank]
    q = hla_synth.attention_inputs_block(B, N, H, d, b0, b1, h0, h1, seed=0)[0]
    # per-rank step time (rank r: r + 1 ms) -> max over ranks; per-rank stats -> all_gather
    m = bch.reduce_max_ms(float(rank + 1), dist, "cpu")
    stats = bch.gather_rank_stats([rank, b0, b1, float(q.float().sum())], dist, "cpu")
    dist.barrier()
    out[rank] = (m, stats, q.shape)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_planner_max_and_gather(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    import hla_synth
    full = hla_synth.attention_inputs(4, 16, 3, 8, seed=0)[0]
    for r in range(world):
        m, stats, shape = res[r]
        assert m == float(world)                                  # max over ranks
        assert len(stats) == world
        assert shape == (4 // world, 16, 3, 8)
        for rr, (rk, b0, b1, qsum) in enumerate(stats):           # every rank sees every rank's stats
            assert int(rk) == rr
            assert qsum == pytest.approx(float(full[int(b0):int(b1)].float().sum()))   # its shard of the global batch


def test_gpus_flag_must_match_world(monkeypatch):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("LOCAL_RANK", "0")
    args = bench.parse(["--gpus", "4"])
    with pytest.raises(SystemExit):
        bench._init_dist(args)
