"""Data-parallel host logic on CPU (gloo, world_size 2): contiguous series shards and the
post-compute gather (paper_0911_4498_b200.parallel).  The per-series compute here is the
oracle standing in for ssa_decompose (no GPU in this container); the point is that the
sharded run reproduces the single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_0911_4498_b200.parallel import gather_rows, shard_range


def test_shard_range_partitions():
    for B in (0, 1, 5, 4096, 4097):
        for P in (1, 2, 3, 8):
            seen = []
            for r in range(P):
                a, b = shard_range(B, r, P)
                assert 0 <= a <= b <= B
                seen.extend(range(a, b))
            assert seen == list(range(B))
            sizes = [shard_range(B, r, P)[1] - shard_range(B, r, P)[0] for r in range(P)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _series(i, N):
    rng = np.random.default_rng([77, i])
    n = np.arange(1, N + 1)
    return np.sin(2 * np.pi * n / 7.5) + 0.3 * rng.standard_normal(N)


def _worker(rank, world, port, B, N, L, k, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    a, b = shard_range(B, rank, world)
    sig = np.stack([oracle.svd(_series(i, N), L, k)[0] for i in range(a, b)]) if b > a else np.zeros((0, k))
    allsig = gather_rows(torch.from_numpy(sig), world)
    if rank == 0:
        np.save(out, allsig.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_equals_single_process(tmp_path):
    import oracle
    B, N, L, k = 7, 24, 10, 3
    out = str(tmp_path / "sig.npy")
    mp.spawn(_worker, args=(2, _free_port(), B, N, L, k, out), nprocs=2, join=True)
    got = np.load(out)
    ref = np.stack([oracle.svd(_series(i, N), L, k)[0] for i in range(B)])
    assert got.shape == ref.shape and np.array_equal(got, ref)
