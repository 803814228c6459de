"""Multi-GPU plumbing: one process per GPU, particles sharded contiguously per group
(ff_set_shard / ff_shard_range), and the path's one exchange step -- the per-frame sum of the
int32 density images -- as a torch.distributed all-reduce (NCCL over NVLink/NVSwitch on GPUs, gloo
on CPU in the tests). Parameters changed on rank 0 are broadcast so every shard integrates the
same system."""
import os

import torch
import torch.distributed as dist

from .fireflies import ff_shard_range  # noqa: F401  (re-exported: the sharding rule)


def init_from_env(backend=None):
    """Initialise the default process group from torchrun's env (RANK, WORLD_SIZE, MASTER_*)."""
    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world


def reduce_image(image, to_rank=None, group=None):
    """Sum the per-rank int32 images in place (all ranks, or only `to_rank`). Integer sums are
    associative, so the result is bit-identical to the unsharded image."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return image
    if to_rank is None:
        dist.all_reduce(image, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.reduce(image, dst=to_rank, op=dist.ReduceOp.SUM, group=group)
    return image


def broadcast_params(ctx, names, src=0, device=None):
    """Broadcast the current values of `names` from rank `src` and apply them with ff_set_param."""
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return
    vals = torch.tensor([ctx.get_param(n) for n in names], dtype=torch.float32, device=device)
    dist.broadcast(vals, src=src)
    for n, v in zip(names, vals.tolist()):
        ctx.set_param(n, v)
