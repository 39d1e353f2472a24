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


def _record_worker(rank, world, port, total, out):
    """Each rank builds result-shaped records for its shard — q (float64),
    losses (float64, including non-finite values of a failed candidate) and an
    int32 status word with high bits set — and gathers them like bench.py."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard.shard_range(total, world, rank)
    rng = np.random.default_rng(lo)
    q = rng.normal(size=(hi - lo, 16))
    losses = rng.normal(size=(hi - lo, 3))
    status = (np.arange(lo, hi, dtype=np.int64) * 2654435761 % (1 << 31)).astype(np.int32)
    if lo <= 3 < hi:
        losses[3 - lo] = [np.nan, np.inf, -np.inf]
    rec = np.concatenate([q, status[:, None].astype(np.float64), losses], axis=1)
    full = shard.gather_rows(rec, total, world, rank)
    if rank == 0:
        np.save(out, full)
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [9, 64])
def test_two_rank_gather_result_records(tmp_path, total):
    out = str(tmp_path / "rec.npy")
    mp.spawn(_record_worker, args=(2, _free_port(), total, out), nprocs=2, join=True)
    full = np.load(out)
    assert full.shape == (total, 20)
    for lo, hi in (shard.shard_range(total, 2, r) for r in range(2)):
        rng = np.random.default_rng(lo)
        assert np.array_equal(full[lo:hi, :16], rng.normal(size=(hi - lo, 16)))
        want_l = rng.normal(size=(hi - lo, 3))
        if lo <= 3 < hi:
            want_l[3 - lo] = [np.nan, np.inf, -np.inf]
        assert np.array_equal(full[lo:hi, 17:], want_l, equal_nan=True)
    status = full[:, 16].astype(np.int64).astype(np.int32)
    want = (np.arange(total, dtype=np.int64) * 2654435761 % (1 << 31)).astype(np.int32)
    assert np.array_equal(status, want)  # every status bit survives the float64 gather exactly


def test_object_major_covers_every_object_once():
    for world in (1, 2, 4, 8):
        objs = [o for r in range(world) for o, _, _ in shard.object_major(64, 1024, world, r)]
        assert objs == list(range(64))


def test_bench_refuses_missing_gpus():
    """`bench.py --gpus 2` without a launcher spawns one rank per GPU, and with
    fewer GPUs visible (this CPU box: none) exits non-zero instead of quietly
    running one rank."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0
    assert "requested but 0 CUDA device" in r.stderr
    assert '"n_gpus"' not in r.stdout
