"""The NVLS variant of the image exchange (ff_set_exchange_multicast): two
processes on two GPUs, images in torch symmetric memory, the sum pass through NVSwitch multicast
(multimem.ld_reduce + multimem.st), or the histogram's reductions as multimem.red (push). Each rank's image must equal the oracle histogram of all particles
(bin-only frame) and the unsharded single-process image (integrating frames), bit-exact. Needs >= 2
GPUs on a multicast-capable NVSwitch system: skipped otherwise (the one-GPU boxes of this run refuse
multicast objects, tools/probe_mc.py)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

from test_gpu_exchange_mp import AXES, GROUPS, LO, HI, SHAPE, VIEW, free_port, make_ctx  # noqa: E402


def worker(rank, world, port, out, push=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_1505_00344_b200 import dist as ffdist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    ctx = make_ctx(rank, world)
    C_, H, W = SHAPE
    try:
        img = ffdist.bind_exchanged_image(ctx, AXES, VIEW, W, H, C_, timeout_ms=30000.0, mapping="symmetric",
                                          multicast=True, push=push)
    except RuntimeError as e:
        out[rank] = f"skip: {e}"
        dist.destroy_process_group()
        return
    frames = []
    for n_steps in (0, 4, 7):
        img.zero_()
        ctx.step(n_steps, 0.01)
        ctx.sync()
        frames.append(img.cpu().numpy().view(np.uint32).copy())
        dist.barrier()
    out[rank] = frames
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("push", [False, True])
def test_nvls_exchange_matches_oracle_and_unsharded_run(push):
    """push=False: the sum pass through multimem.ld_reduce / multimem.st; push=True: the histogram's
    reductions issued once each as multimem.red.add to the multicast address (ff_set_exchange_push)."""
    import torch.multiprocessing as mp
    import oracle as O
    world = 2
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(worker, args=(world, free_port(), out, push), nprocs=world, join=True)
    if any(isinstance(out[r], str) for r in range(world)):
        pytest.skip(str(out[0]))
    C_, H, W = SHAPE
    want0 = np.zeros(SHAPE, np.uint32)
    for n, seed, _, colour in GROUPS:
        O.histogram(O.ic_uniform(LO, HI, seed, 0, n), AXES, VIEW, W, H, C_, colour, image=want0)
    ctx = make_ctx(0, 1)
    img = ctx.project(AXES, VIEW, W, H, C_)
    plain = []
    for n_steps in (0, 4, 7):
        img.zero_()
        ctx.step(n_steps, 0.01)
        plain.append(ctx.read_image())
    assert np.array_equal(plain[0], want0)
    for rank in range(world):
        for f in range(3):
            assert np.array_equal(out[rank][f], plain[f]), (rank, f)
