"""The image exchange across PROCESSES (one GPU, two ranks): dist.bind_exchanged_image maps the
peers' images with CUDA IPC (torch symmetric memory refuses two ranks on one device; across GPUs the
same code maps NVLink peer memory), ff_set_exchange sums them after every binning launch (or, with
ff_set_exchange_push, the histogram's reductions go to both images). Each rank's
image must equal the oracle histogram of all particles (bin-only frame) and the unsharded image of a
single-process run (integrating frames), bit-exact."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

LO, HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]
GROUPS = [(30011, 2, 1, 0), (20003, 3, -1, 1)]      # (n, seed, direction, colour)
AXES, VIEW, SHAPE = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 61, 83)   # ragged: C*H*W % 4 = 2


def make_ctx(rank, world):
    import paper_1505_00344_b200 as FF
    from paper_1505_00344_b200 import systems
    ctx = FF.Context(systems.lorenz(), [n for n, _, _, _ in GROUPS], rank=rank, world=world)
    for n, seed, d, colour in GROUPS:
        ctx.init_group(LO, HI, n, d, colour, seed)
    return ctx


def worker(rank, world, port, out, push=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_1505_00344_b200 import dist as ffdist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    ctx = make_ctx(rank, world)
    C_, H, W = SHAPE
    img = ffdist.bind_exchanged_image(ctx, AXES, VIEW, W, H, C_, timeout_ms=30000.0, mapping="ipc", push=push)
    frames = []
    for n_steps in (0, 4, 7):
        img.zero_()
        ctx.step(n_steps, 0.01)
        ctx.sync()
        frames.append(img.cpu().numpy().view(np.uint32).copy())
        dist.barrier()                   # nobody zeroes its image while a peer still reads it
    out[rank] = frames
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("push", [False, True])
def test_two_process_exchange_matches_oracle_and_unsharded_run(push):
    """push=False: the sum pass after each launch (ff_set_exchange); push=True: the histogram's
    reductions sent to both processes' images (ff_set_exchange_push, red.add over the IPC mapping)."""
    import torch.multiprocessing as mp
    import oracle as O
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(worker, args=(world, free_port(), out, push), nprocs=world, join=True)
    C_, H, W = SHAPE
    want0 = np.zeros(SHAPE, np.uint32)
    for n, seed, _, colour in GROUPS:
        O.histogram(O.ic_uniform(LO, HI, seed, 0, n), AXES, VIEW, W, H, C_, colour, image=want0)
    ctx = make_ctx(0, 1)               # the unsharded single-process run
    img = ctx.project(AXES, VIEW, W, H, C_)
    plain = []
    for n_steps in (0, 4, 7):
        img.zero_()
        ctx.step(n_steps, 0.01)
        plain.append(ctx.read_image())
    assert np.array_equal(plain[0], want0) and want0.sum() > 0
    for rank in range(world):
        for f in range(3):
            assert np.array_equal(out[rank][f], plain[f]), (rank, f)
