"""Multi-GPU plumbing: one process per GPU, particles sharded contiguously per group
(ff_set_shard / ff_shard_range), and the path's one exchange step -- the per-frame sum of the
int32 density images -- either fused into the step launch over NVLink peer memory
(bind_exchanged_image -> ff_set_exchange: a sum pass after the launch, or with push=True the
histogram's own reductions sent to every rank's image, ff_set_exchange_push; torch symmetric memory
only maps the buffers) or as a
torch.distributed all-reduce (reduce_image: NCCL over NVLink/NVSwitch on GPUs, gloo on CPU in the
tests). Parameters changed on rank 0 are broadcast so every shard integrates the same system
(PAPER.md:242)."""
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


FF_MAX_PEERS = 8


def exchange_layout(C_, H, W):
    """Symmetric buffer layout of one rank for the fused exchange, in int32 words: the image
    [C][H][W] first, then FF_MAX_PEERS uint64 signal words at a 256-byte boundary.
    Returns (image_words, signal_offset_bytes, total_words)."""
    words = int(C_) * int(H) * int(W)
    sig_words = (words + 63) // 64 * 64
    return words, 4 * sig_words, sig_words + 2 * FF_MAX_PEERS


def peer_tables(buffer_ptrs, C_, H, W):
    """(peer image pointers, peer signal pointers) from every rank's symmetric buffer base address."""
    _, sig_off, _ = exchange_layout(C_, H, W)
    return [int(p) for p in buffer_ptrs], [int(p) + sig_off for p in buffer_ptrs]


def _map_symmetric(buf, group):
    """torch symmetric memory: (buffer pointers of every rank, rank, world, keepalive)."""
    import torch.distributed._symmetric_memory as symm_mem
    handle = symm_mem.rendezvous(buf, group)
    return list(handle.buffer_ptrs), handle.rank, handle.world_size, handle


def _map_ipc(buf, group):
    """CUDA IPC (the mechanism torch.multiprocessing uses for CUDA tensors): every rank exports its
    buffer, opens the others'. Works across GPUs with peer access and between processes sharing one
    GPU (where torch symmetric memory refuses). Returns the same tuple as _map_symmetric."""
    from torch.multiprocessing.reductions import reduce_tensor
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    rebuild, args = reduce_tensor(buf)
    shared = [None] * world
    dist.all_gather_object(shared, (rebuild, args), group=group)
    peers = [buf if r == rank else fn(*a) for r, (fn, a) in enumerate(shared)]
    return [t.data_ptr() for t in peers], rank, world, peers


def bind_exchanged_image(ctx, axes, view, W, H, C_=1, group=None, timeout_ms=1000.0, mapping="auto",
                         multicast=False, push=False):
    """Bind a peer-accessible image to `ctx` and turn on the library's image exchange: from now on
    every binning ff_step of every rank is followed, on its stream, by the sum of the images over all
    ranks (ff_set_exchange; no separate collective). Collective over `group` (default: the world);
    returns the bound image tensor [C][H][W] (int32, zeroed). mapping: "symmetric" (torch symmetric
    memory), "ipc" (CUDA IPC handles), "auto" (symmetric, else IPC). multicast=True additionally binds
    the NVLS multicast mapping of the images (torch symmetric memory's multicast_ptr;
    ff_set_exchange_multicast) and raises if the system offers none. push=True selects the fused
    (push) exchange instead of the sum pass: the histogram's reductions go straight to every rank's
    image (over peer memory, or with multicast=True as multimem.red through the multicast mapping;
    ff_set_exchange_push) between two barriers per launch; zero the image on every rank per frame."""
    words, sig_off, total = exchange_layout(C_, H, W)
    if not dist.is_initialized() or dist.get_world_size(group) == 1:   # one rank: its own tables
        buf = torch.zeros(total, dtype=torch.int32, device=ctx.device)
        image = buf[:words].view(C_, H, W)
        ctx.project(axes, view, W, H, C_, image=image)
        image.zero_()
        torch.cuda.synchronize(ctx.device)
        imgs, sigs = peer_tables([buf.data_ptr()], C_, H, W)
        ctx.set_exchange(0, 1, imgs, sigs, timeout_ms)
        if push:
            ctx.set_exchange_push(True)
        ctx._symm = (buf,)
        return image
    group = group if group is not None else dist.group.WORLD
    mapped = None
    if mapping in ("auto", "symmetric"):
        try:
            import torch.distributed._symmetric_memory as symm_mem
            buf = symm_mem.empty(total, dtype=torch.int32, device=ctx.device)
            buf.zero_()
            mapped = _map_symmetric(buf, group)
        except Exception:   # (no symmetric-memory backend for this group / same-device ranks)
            if mapping == "symmetric":
                raise
            mapped = None
    if mapped is None:
        buf = torch.zeros(total, dtype=torch.int32, device=ctx.device)
        torch.cuda.synchronize(ctx.device)
        mapped = _map_ipc(buf, group)
    ptrs, rank, world, keep = mapped
    image = buf[:words].view(C_, H, W)
    ctx.project(axes, view, W, H, C_, image=image)   # binds (and bins the current state locally)
    image.zero_()
    buf[words:].zero_()
    torch.cuda.synchronize(ctx.device)
    dist.barrier(group)                                # every rank's signals are zero
    imgs, sigs = peer_tables(ptrs, C_, H, W)
    ctx.set_exchange(rank, world, imgs, sigs, timeout_ms)
    if multicast:
        mc = int(getattr(keep, "multicast_ptr", 0) or 0)
        ok = torch.tensor([1 if mc else 0], dtype=torch.int32, device=ctx.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)   # all ranks or none
        if not int(ok.item()):
            ctx.set_exchange(0, 0)
            raise RuntimeError("no NVLS multicast mapping for this group (symmetric memory multicast_ptr = 0)")
        if push:
            ctx.set_exchange_push(True, mc)
        else:
            ctx.set_exchange_multicast(mc)
    elif push:
        ctx.set_exchange_push(True)
    ctx._symm = (buf, keep)                            # keep the mappings alive with the context
    return image
