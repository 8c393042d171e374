"""Multi-rank host logic on CPU (gloo, world_size 2): the batch split covers every trace exactly
once, each rank's shard transformed independently (here by the CPU oracle — the data path has
no collective) and gathered equals the single-rank result bit for bit."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_03948_b200.sharding import gather_rows, shard_bounds


def test_shard_bounds_cover_batch():
    for batch in (0, 1, 7, 8192, 8193):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _worker(rank, world, port, batch, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    from paper_2108_03948_b200 import workloads as W
    x = W.cfg2_batch(7, 256)[:batch]
    a, w = W.cfg2_czt_params(200)
    b0, b1 = shard_bounds(x.shape[0], rank, world)
    local = torch.from_numpy(O.CztPlan(256, a, w, 200).batch_real(x[b0:b1]))
    full = gather_rows(local, x.shape[0])
    if rank == 0:
        np.save(out, full.numpy())
    dist.destroy_process_group()


def test_two_rank_shard_and_gather(tmp_path):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "full.npy")
    batch = 13   # uneven: 7 + 6 rows
    mp.spawn(_worker, args=(2, port, batch, out), nprocs=2, join=True)
    import oracle as O
    from paper_2108_03948_b200 import workloads as W
    x = W.cfg2_batch(7, 256)[:batch]
    a, w = W.cfg2_czt_params(200)
    want = O.CztPlan(256, a, w, 200).batch_real(x)
    np.testing.assert_array_equal(np.load(out), want)
