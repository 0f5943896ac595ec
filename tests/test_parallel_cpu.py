"""Multi-process host logic of the sharded driver on CPU (gloo, world_size 2): the
partitioner covers every image exactly once in order, the metadata all_gather returns
every rank's [count, elapsed, checksum], and concatenating per-rank outputs of an
image-independent map equals the single-process result (the shard-invariance the GPU
test checks bitwise on the real kernels)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2210_08650_b200.parallel import checksum_bits, gather_meta, run_shard, shard_range, summarize


@pytest.mark.parametrize("n,world", [(0, 1), (7, 1), (7, 2), (65536, 8), (513, 4), (3, 8)])
def test_shard_range_partition(n, world):
    got = [shard_range(n, world, r) for r in range(world)]
    assert got[0][0] == 0 and got[-1][1] == n
    for (a0, b0), (a1, b1) in zip(got, got[1:]):
        assert b0 == a1 and a0 <= b0
    sizes = [b - a for a, b in got]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_errors():
    for args in [(5, 0, 0), (5, 2, 2), (5, 2, -1), (-1, 1, 0)]:
        with pytest.raises(ValueError):
            shard_range(*args)


def test_checksum_bits_roundtrip():
    for x in [0.0, -1.5, 955379584.0, 1e-300]:
        assert float(np.int64(checksum_bits(x)).view(np.float64)) == x


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    data = np.arange(n, dtype=np.float64) * 0.5
    outs = []

    def fwd(start, count):  # an image-independent stand-in for the prefix forward
        y = np.sqrt(data[start:start + count]) + 1.0
        outs.append((start, y))
        return float(y.sum())

    count, cks = run_shard(n, world, rank, 3, fwd)
    meta = gather_meta(count, 1000 * (rank + 1), cks)
    q.put((rank, meta.tolist(), [(s, y.tolist()) for s, y in outs]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_gather_and_shard_invariance():
    world, n = 2, 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    metas = [np.array(m, dtype=np.int64) for _, m, _ in res]
    np.testing.assert_array_equal(metas[0], metas[1])  # every rank sees every rank's meta
    total, tmax, rate, checks = summarize(metas[0])
    assert total == n and tmax == 2000 / 1e9
    # concatenation of per-rank chunks in rank order == single-process map
    pieces = sorted(((s, y) for _, _, outs in res for s, y in outs), key=lambda t: t[0])
    cat = np.concatenate([np.array(y) for _, y in pieces])
    np.testing.assert_array_equal(cat, np.sqrt(np.arange(n) * 0.5) + 1.0)
    assert abs(sum(checks) - cat.sum()) < 1e-9
