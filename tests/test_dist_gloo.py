"""Multi-process host logic of the multi-GPU path on CPU (gloo, world size 2): the library's shard
rule (ff_shard_range) + dist.reduce_image summing per-rank images gives exactly the unsharded image,
and dist.broadcast_params propagates rank 0's parameter values."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

LO, HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]
P = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
GROUPS = [(1001, 2, 0.01, 0), (777, 3, -0.01, 1)]   # (n, seed, h, colour)
VIEW = [-20.0, 20.0, -30.0, 30.0]


def shard_image(rank, world):
    from paper_1505_00344_b200.fireflies import ff_shard_range
    img = np.zeros((2, 32, 48), np.uint32)
    for n, seed, h, colour in GROUPS:
        first, count = ff_shard_range(n, rank, world)
        x = O.ic_uniform(LO, HI, seed, first, count)
        x = O.rk4(O.LORENZ, x, P, np.float32(h), 5)
        O.histogram(x, [0, 1], VIEW, 48, 32, 2, colour, image=img)
    return img


class FakeCtx:
    def __init__(self, v):
        self.v = {"r": v}

    def get_param(self, k):
        return self.v[k]

    def set_param(self, k, v):
        self.v[k] = v


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_1505_00344_b200 import dist as ffdist
    r, w = ffdist.init_from_env("gloo")
    assert (r, w) == (rank, world)
    img = torch.from_numpy(shard_image(rank, world).astype(np.int32))
    ffdist.reduce_image(img)
    ctx = FakeCtx(28.0 if rank == 0 else -1.0)
    ffdist.broadcast_params(ctx, ["r"])
    out[rank] = (img.numpy().copy(), ctx.v["r"])
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_images_reduce_to_unsharded_image():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    whole = shard_image(0, 1).astype(np.int32)
    for rank in range(world):
        img, r = out[rank]
        assert np.array_equal(img, whole)
        assert r == 28.0
    assert whole.sum() > 0


def test_shard_ranges_partition_every_group():
    from paper_1505_00344_b200.fireflies import ff_shard_range
    for n in (1, 7, 1000, 2 ** 30 + 3):
        for world in (1, 2, 3, 8):
            parts = [ff_shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0
            for (f0, c0), (f1, _) in zip(parts, parts[1:]):
                assert f0 + c0 == f1
            assert parts[-1][0] + parts[-1][1] == n
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1


def _exchange_worker(rank, world, port, out):
    """Host side of the fused exchange (bind_exchanged_image): every rank derives identical peer
    tables from the gathered symmetric-buffer bases (fake addresses here: no GPU)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_1505_00344_b200 import dist as ffdist
    ffdist.init_from_env("gloo")
    bases = [None] * world
    dist.all_gather_object(bases, 0x7f0000000000 + rank * (1 << 30))
    out[rank] = ffdist.peer_tables(bases, 2, 29, 37)
    dist.barrier()
    dist.destroy_process_group()


def test_exchange_peer_tables_agree_across_ranks():
    from paper_1505_00344_b200 import dist as ffdist
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_exchange_worker, args=(world, free_port(), out), nprocs=world, join=True)
    assert out[0] == out[1]
    imgs, sigs = out[0]
    words, sig_off, total = ffdist.exchange_layout(2, 29, 37)
    for i, s in zip(imgs, sigs):
        assert i % 256 == 0 and (s - i) == sig_off and sig_off % 256 == 0
        assert sig_off >= 4 * words and 4 * total - sig_off == 8 * ffdist.FF_MAX_PEERS
