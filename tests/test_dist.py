"""N>1 path on CPU: world_size-2 gloo processes shard a batch with the
library's shard rule (xlf_shard, which bench.py and the MultiEngine use: rank
r owns images [r*B, (r+1)*B) of the seeded stream), compute their shard
independently (the CPU oracle stands in for the device: no GPU here; no
exchange on the data path) and gather to rank 0; the result must equal the
single-process run bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, out_path):
    import torch
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2007_06000_b200 import dist as D
    from paper_2007_06000_b200 import graph_path
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    og = O.load_graph(open(graph_path("a1")).read())
    w = O.seeded_weights(og, 42)
    first, count = D.shard(rank, world, per_rank)
    c, h, wd = og.inputs[0][1]
    x = O.stream(42, first * c * h * wd, count * c * h * wd).reshape(count, c, h, wd)
    y = O.run_batch(og, x, w, ["conv2"])["conv2"]
    t = D.max_over_ranks(float(rank + 1))
    assert t == float(world)
    g = D.gather_to_rank0(torch.from_numpy(y))
    if rank == 0:
        np.save(out_path, g.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_batch_sharding_gloo(tmp_path, world):
    from oracle import oracle as O
    from paper_2007_06000_b200 import graph_path
    per_rank = 2
    out = str(tmp_path / "g.npy")
    mp.start_processes(_worker, args=(world, _free_port(), per_rank, out), nprocs=world, start_method="spawn")
    got = np.load(out)
    og = O.load_graph(open(graph_path("a1")).read())
    x = O.seeded_batch(og, 42, world * per_rank)
    ref = O.run_batch(og, x, O.seeded_weights(og, 42), ["conv2"])["conv2"]
    assert got.shape == ref.shape and np.array_equal(got, ref)


def test_library_shard_rule_ragged():
    """xlf_shard (the MultiEngine's rule): contiguous, sizes differ by <= 1."""
    from paper_2007_06000_b200 import shard_range
    for batch in (0, 1, 5, 7, 255, 256, 2048):
        for n in (1, 2, 3, 4, 8):
            ranges = [shard_range(batch, n, k) for k in range(n)]
            seen = [i for f, c in ranges for i in range(f, f + c)]
            assert seen == list(range(batch))
            assert max(c for _, c in ranges) - min(c for _, c in ranges) <= 1


def test_shard_covers_batch_once():
    from paper_2007_06000_b200 import dist as D
    for world in (1, 2, 4, 8):
        seen = []
        for r in range(world):
            f, n = D.shard(r, world, 256)
            seen += list(range(f, f + n))
        assert seen == list(range(256 * world))
    with pytest.raises(ValueError):
        D.shard(2, 2, 1)
