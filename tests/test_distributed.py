"""Multi-process (world_size 2, gloo on CPU) coverage of the env-sharded
N>1 path: slices, per-shard commands, max-over-ranks timing, rollout-stat
gather. The step itself has no collective."""
import os
import socket

import numpy as np
import pytest

from paper_1904_02833_b200.distributed import env_slice


def test_env_slices_partition():
    for total in (1, 7, 1024, 65536):
        for world in (1, 2, 3, 8):
            got = [env_slice(total, world, r) for r in range(world)]
            assert got[0][0] == 0
            for (a0, n0), (a1, _) in zip(got, got[1:]):
                assert a0 + n0 == a1
            assert sum(n for _, n in got) == total
            assert max(n for _, n in got) - min(n for _, n in got) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from paper_1904_02833_b200.distributed import (env_slice, gather_env_stats,
                                                       max_over_ranks)
        env0, n = env_slice(total, world, rank)
        cmds = bench.env_commands(n, 3, 0, env0=env0)
        stats = np.stack([np.arange(env0, env0 + n, dtype=float), cmds[0, :, 0]], axis=1)
        allstats = gather_env_stats(stats, total)
        t = max_over_ranks(float(rank + 1))
        q.put((rank, allstats, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_gather_and_max():
    import multiprocessing as mp
    import bench
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    total, world, port = 11, 2, _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    full = bench.env_commands(total, 3, 0)
    for rank, allstats, t in res:
        assert t == 2.0                                   # max over ranks
        assert np.array_equal(allstats[:, 0], np.arange(total))
        assert np.array_equal(allstats[:, 1], full[0, :, 0])  # shard commands == global slice
