"""CPU, multi-process (gloo, world_size 2): candidate sharding and the final
gather reproduce the single-process batch exactly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2306_08132_b200 import shard


def test_shard_range_partition():
    for total in (0, 1, 7, 1024, 1025):
        for world in (1, 2, 3, 8):
            got = [shard.shard_range(total, world, r) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(h - l for l, h in got) - min(h - l for l, h in got) <= 1
    assert shard.object_major(64, 1024, 8, 3) == [(o, 0, 1024) for o in range(24, 32)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out):
    import torch.distributed as dist
    from paper_2306_08132_b200 import init, model
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hand = model.HandDesc.asset("barrett3")
    obj = model.sphere(0.025)
    lo, hi = shard.shard_range(total, world, rank)
    q = init.approach_init(obj, hand, hi - lo, seed=3, first=lo)  # shard-local init, global indices
    rec = np.concatenate([q, np.arange(lo, hi, dtype=np.float64)[:, None]], axis=1)
    full = shard.gather_rows(rec, total, world, rank)
    if rank == 0:
        np.save(out, full)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [10, 33])
def test_two_rank_gather_matches_single_process(tmp_path, total):
    from paper_2306_08132_b200 import init, model
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(2, _free_port(), total, out), nprocs=2, join=True)
    full = np.load(out)
    hand = model.HandDesc.asset("barrett3")
    ref = init.approach_init(model.sphere(0.025), hand, total, seed=3)
    assert np.array_equal(full[:, :-1], ref)
    assert np.array_equal(full[:, -1], np.arange(total))
