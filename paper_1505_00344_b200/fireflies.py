"""Thin Python binding of libfireflies (include/fireflies.h).

Functions named ff_* are one-to-one wrappers of the C ABI (marshalling only). `Context` is
plumbing on top: it owns the torch tensors that hold the caller-owned device memory (particle state
[dim][pitch] and the density image [C][H][W]) and passes torch's current stream. Every step of the
hot path runs in the library's kernels; nothing here computes.
"""
import ctypes as C

import numpy as np

from . import _abi
from ._abi import FF_TILE, FFError, check, lib, make_system  # noqa: F401
from .systems import SystemDef


def _fptr(a):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------- one-to-one C ABI wrappers
def ff_last_error() -> str:
    return lib().ff_last_error().decode()


def ff_abi_version() -> int:
    return lib().ff_abi_version()


def ff_build_info() -> str:
    buf = C.create_string_buffer(1024)
    check(lib().ff_build_info(buf, 1024, None))
    return buf.value.decode()


def ff_emit_source(system: SystemDef, sweep_param: int = -1) -> str:
    s, keep = make_system(system.var_names, system.rhs, system.params)
    n = C.c_size_t(0)
    check(lib().ff_emit_source(C.byref(s), sweep_param, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    check(lib().ff_emit_source(C.byref(s), sweep_param, buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def ff_compile_cubin(system: SystemDef, sweep_param: int = -1) -> bytes:
    s, keep = make_system(system.var_names, system.rhs, system.params)
    n = C.c_size_t(0)
    check(lib().ff_compile_cubin(C.byref(s), sweep_param, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value)
    check(lib().ff_compile_cubin(C.byref(s), sweep_param, buf, n.value, C.byref(n)))
    return buf.raw[:n.value]


def ff_create(system: SystemDef, device: int = 0) -> C.c_void_p:
    s, keep = make_system(system.var_names, system.rhs, system.params)
    ctx = C.c_void_p()
    check(lib().ff_create(C.byref(s), device, C.byref(ctx)))
    return ctx


def ff_destroy(ctx):
    check(lib().ff_destroy(ctx))


def ff_set_stream(ctx, stream_handle: int):
    check(lib().ff_set_stream(ctx, C.c_void_p(stream_handle)))


def ff_set_shard(ctx, rank: int, world: int):
    check(lib().ff_set_shard(ctx, rank, world))


def ff_shard_range(n_global: int, rank: int, world: int):
    first, count = C.c_int64(), C.c_int64()
    check(lib().ff_shard_range(n_global, rank, world, C.byref(first), C.byref(count)))
    return first.value, count.value


def ff_bind_state(ctx, dev_ptr: int, pitch: int, capacity: int):
    check(lib().ff_bind_state(ctx, C.c_void_p(dev_ptr), pitch, capacity))


def ff_group_slots(ctx, n_global: int) -> int:
    out = C.c_int64()
    check(lib().ff_group_slots(ctx, n_global, C.byref(out)))
    return out.value


def ff_init_group(ctx, ic_lo, ic_hi, n_global: int, direction: int, colour: int, seed: int) -> int:
    lo = np.ascontiguousarray(ic_lo, dtype=np.float32)
    hi = np.ascontiguousarray(ic_hi, dtype=np.float32)
    gid = C.c_int(-1)
    check(lib().ff_init_group(ctx, _fptr(lo), _fptr(hi), n_global, direction, colour, seed, C.byref(gid)))
    return gid.value


def ff_group_info(ctx, group_id: int):
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().ff_group_info(ctx, group_id, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, c.value


def ff_set_param(ctx, name: str, value: float):
    check(lib().ff_set_param(ctx, name.encode(), value))


def ff_get_param(ctx, name: str) -> float:
    v = C.c_float()
    check(lib().ff_get_param(ctx, name.encode(), C.byref(v)))
    return v.value


def ff_sweep_param(ctx, group_id: int, name: str, lo: float, hi: float, mode: int = 0, seed: int = 0):
    check(lib().ff_sweep_param(ctx, group_id, name.encode(), lo, hi, mode, seed))


def ff_project(ctx, axes, view, W: int, H: int, C_: int, dev_image_ptr):
    ax = np.ascontiguousarray(axes, dtype=np.int32)
    vw = np.ascontiguousarray(view, dtype=np.float32).ravel()
    check(lib().ff_project(ctx, _fptr(ax), ax.size, _fptr(vw), W, H, C_,
                           C.c_void_p(dev_image_ptr) if dev_image_ptr else None))


def ff_step(ctx, n_steps: int, dt: float):
    check(lib().ff_step(ctx, n_steps, dt))


def ff_set_reset(ctx, enable: bool, lo=None, hi=None, t_max: float = 0.0):
    lo_a = None if lo is None else np.ascontiguousarray(lo, dtype=np.float32)
    hi_a = None if hi is None else np.ascontiguousarray(hi, dtype=np.float32)
    check(lib().ff_set_reset(ctx, 1 if enable else 0, None if lo_a is None else _fptr(lo_a),
                             None if hi_a is None else _fptr(hi_a), t_max))


def ff_read_epochs(ctx, group_id: int, first: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint32)
    check(lib().ff_read_epochs(ctx, group_id, first, count, _fptr(out)))
    return out


def ff_read_lifted(ctx, group_id: int, first: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float32)
    check(lib().ff_read_lifted(ctx, group_id, first, count, _fptr(out)))
    return out


def ff_set_launch(ctx, particles_per_thread: int = 0, threads_per_block: int = 0):
    check(lib().ff_set_launch(ctx, particles_per_thread, threads_per_block))


def ff_read_state(ctx, group_id: int, first: int, count: int, dim: int) -> np.ndarray:
    out = np.empty((dim, count), dtype=np.float32)
    check(lib().ff_read_state(ctx, group_id, first, count, _fptr(out)))
    return out


def ff_write_state(ctx, group_id: int, first: int, host_soa, dim: int) -> None:
    a = np.ascontiguousarray(host_soa, dtype=np.float32)
    # the library copies dim rows of a.shape[1] floats from this buffer: the shape must be (dim, count)
    if a.ndim != 2 or a.shape[0] != dim:
        raise ValueError(f"host_soa must have shape (dim={dim}, count), got {a.shape}")
    check(lib().ff_write_state(ctx, group_id, first, a.shape[1], _fptr(a)))


def ff_read_image_into(ctx, host_ptr: int):
    check(lib().ff_read_image(ctx, C.c_void_p(host_ptr)))


def ff_write_state_async(ctx, group_id: int, first: int, count: int, host_ptr: int):
    """Stream-ordered copy-in of [dim][count] floats from (pinned) host memory at host_ptr."""
    check(lib().ff_write_state_async(ctx, group_id, first, count, C.c_void_p(host_ptr)))


def ff_read_image_async(ctx, host_ptr: int):
    """Stream-ordered copy-out of the bound image to (pinned) host memory at host_ptr."""
    check(lib().ff_read_image_async(ctx, C.c_void_p(host_ptr)))


def ff_render(ctx, colours, intensity: float, radius_px: float, dev_rgb_ptr: int):
    col = np.ascontiguousarray(colours, dtype=np.float32)
    check(lib().ff_render(ctx, _fptr(col), intensity, radius_px, C.c_void_p(dev_rgb_ptr)))


def ff_launch_count(ctx) -> int:
    n = C.c_int64()
    check(lib().ff_launch_count(ctx, C.byref(n)))
    return n.value


def ff_sync(ctx):
    check(lib().ff_sync(ctx))


def ff_set_exchange(ctx, rank: int, world: int, peer_image_ptrs, peer_signal_ptrs, timeout_ms: float = 1000.0):
    """Fused in-launch image all-reduce over peer memory (world = 0: off). Pointers are ints."""
    if world == 0:
        check(lib().ff_set_exchange(ctx, 0, 0, None, None, 1.0))
        return
    imgs = (C.c_void_p * world)(*[int(p) for p in peer_image_ptrs])
    sigs = (C.c_void_p * world)(*[int(p) for p in peer_signal_ptrs])
    check(lib().ff_set_exchange(ctx, rank, world, imgs, sigs, timeout_ms))


def ff_set_exchange_multicast(ctx, mc_image_ptr: int):
    """NVLS multicast address of the exchanged images (0: peer loads / stores)."""
    check(lib().ff_set_exchange_multicast(ctx, C.c_void_p(int(mc_image_ptr)) if mc_image_ptr else None))


def ff_set_exchange_push(ctx, on: bool, mc_image_ptr: int = 0):
    """Fused (push) exchange: the histogram's reductions go to every rank's image (mc_image_ptr = 0:
    red.add per peer image; else multimem.red.add through the multicast address)."""
    check(lib().ff_set_exchange_push(ctx, 1 if on else 0, C.c_void_p(int(mc_image_ptr)) if mc_image_ptr else None))


def ff_set_grid_limit(ctx, max_blocks: int):
    check(lib().ff_set_grid_limit(ctx, max_blocks))


# ---------------------------------------------------------------- plumbing: Context
class Context:
    """One system on one CUDA device (torch for memory and the stream).

    group_sizes: the n_global of every group that will be created (sizes the state tensor).
    rank/world: shard every group over `world` processes.
    """

    def __init__(self, system: SystemDef, group_sizes, device=None, rank=0, world=1, extra_slots=0):
        import torch
        self.torch = torch
        self.system = system
        self.dim = system.dim
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        torch.cuda.set_device(self.device)
        self.ctx = ff_create(system, self.device.index)
        self.stream = torch.cuda.current_stream(self.device)
        ff_set_stream(self.ctx, self.stream.cuda_stream)
        if world > 1:
            ff_set_shard(self.ctx, rank, world)
        slots = sum(ff_group_slots(self.ctx, n) for n in group_sizes) + extra_slots
        self.pitch = max(FF_TILE, (slots + FF_TILE - 1) // FF_TILE * FF_TILE)
        self.state = torch.empty((self.dim, self.pitch), dtype=torch.float32, device=self.device)
        ff_bind_state(self.ctx, self.state.data_ptr(), self.pitch, self.pitch)
        self.image = None
        self.groups = []

    def close(self):
        if self.ctx:
            ff_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_group(self, ic_lo, ic_hi, n, direction=1, colour=0, seed=0) -> int:
        g = ff_init_group(self.ctx, ic_lo, ic_hi, n, direction, colour, seed)
        self.groups.append(g)
        return g

    def group_info(self, g):
        return ff_group_info(self.ctx, g)

    def group_view(self, g):
        """torch view [dim][n_local] of a group's slots (no copy)."""
        s, n, _ = ff_group_info(self.ctx, g)
        return self.state[:, s:s + n]

    def set_param(self, name, value):
        ff_set_param(self.ctx, name, value)

    def get_param(self, name):
        return ff_get_param(self.ctx, name)

    def sweep_param(self, g, name, lo, hi, mode=0, seed=0):
        ff_sweep_param(self.ctx, g, name, lo, hi, mode, seed)

    def project(self, axes, view, W, H, C_=1, image=None):
        """Bind (and zero-allocate if needed) the uint32 image [C][H][W]; bins the current state."""
        torch = self.torch
        if image is None:
            image = torch.zeros((C_, H, W), dtype=torch.int32, device=self.device)
        assert image.dtype == torch.int32 and image.is_contiguous() and tuple(image.shape) == (C_, H, W)
        self.image = image
        ff_project(self.ctx, axes, view, W, H, C_, image.data_ptr())
        return image

    def unbind_image(self):
        ff_project(self.ctx, [0, 0], [0, 1, 0, 1], 1, 1, 1, 0)
        self.image = None

    def step(self, n_steps, dt):
        ff_step(self.ctx, n_steps, dt)

    def capture(self, frame):
        """Record `frame()` -- e.g. `lambda: (img.zero_(), ctx.step(S, dt))` -- into a CUDA graph and
        return the torch.cuda.CUDAGraph; `g.replay()` runs the frame again on torch's current stream
        (SURVEY.md A8). Run the frame once before capturing it (its kernels compile at first use)."""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(self.device)
        side.wait_stream(self.stream)
        with torch.cuda.graph(g, stream=side):
            ff_set_stream(self.ctx, side.cuda_stream)
            try:
                frame()
            finally:
                ff_set_stream(self.ctx, self.stream.cuda_stream)
        return g

    def set_reset(self, enable=True, lo=None, hi=None, t_max=0.0):
        ff_set_reset(self.ctx, enable, lo, hi, t_max)

    def read_epochs(self, g, first=0, count=None):
        _, n, _ = ff_group_info(self.ctx, g)
        count = n - first if count is None else count
        return ff_read_epochs(self.ctx, g, first, count)

    def read_lifted(self, g, first=0, count=None):
        _, n, _ = ff_group_info(self.ctx, g)
        count = n - first if count is None else count
        return ff_read_lifted(self.ctx, g, first, count)

    def set_launch(self, ppt=0, tpb=0):
        ff_set_launch(self.ctx, ppt, tpb)

    def read_state(self, g, first=0, count=None):
        _, n, _ = ff_group_info(self.ctx, g)
        count = n - first if count is None else count
        return ff_read_state(self.ctx, g, first, count, self.dim)

    def write_state(self, g, host_soa, first=0):
        ff_write_state(self.ctx, g, first, host_soa, self.dim)

    def read_image(self):
        """Host copy of the bound image as uint32 (C, H, W)."""
        out = np.empty(tuple(self.image.shape), dtype=np.uint32)
        ff_read_image_into(self.ctx, out.ctypes.data)
        return out

    def project_colour(self, lo, hi, colour_image=None):
        """Bind (zero-allocating if needed) the position-colour sums [3][H][W] (ff_project_colour)."""
        torch = self.torch
        C_, H, W = self.image.shape
        if colour_image is None:
            colour_image = torch.zeros((3, H, W), dtype=torch.int32, device=self.device)
        lo_a = np.ascontiguousarray(lo, dtype=np.float32)
        hi_a = np.ascontiguousarray(hi, dtype=np.float32)
        check(lib().ff_project_colour(self.ctx, _fptr(lo_a), _fptr(hi_a), C.c_void_p(colour_image.data_ptr())))
        self.colour_image = colour_image
        return colour_image

    def render(self, colours, intensity=1.0, radius_px=2.0, out=None):
        """RGB float32 [3][H][W] frame of the bound image (device tensor)."""
        torch = self.torch
        C_, H, W = self.image.shape
        if out is None:
            out = torch.empty((3, H, W), dtype=torch.float32, device=self.device)
        ff_render(self.ctx, colours, intensity, radius_px, out.data_ptr())
        return out

    def set_exchange(self, rank, world, peer_image_ptrs=(), peer_signal_ptrs=(), timeout_ms=1000.0):
        ff_set_exchange(self.ctx, rank, world, peer_image_ptrs, peer_signal_ptrs, timeout_ms)

    def set_exchange_multicast(self, mc_image_ptr):
        ff_set_exchange_multicast(self.ctx, mc_image_ptr)

    def set_exchange_push(self, on=True, mc_image_ptr=0):
        ff_set_exchange_push(self.ctx, on, mc_image_ptr)

    def set_grid_limit(self, max_blocks):
        ff_set_grid_limit(self.ctx, max_blocks)

    def launch_count(self):
        return ff_launch_count(self.ctx)

    def sync(self):
        ff_sync(self.ctx)
