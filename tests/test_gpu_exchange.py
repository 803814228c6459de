"""GPU tests of the fused image exchange (ff_set_exchange, NEXT row 2).

The exchange is the path's one collective -- the per-frame sum of the ranks' density images -- done
by the library over peer memory in a kernel that follows each binning launch. This box has one GPU,
so several ranks are emulated by several contexts sharing it: each context integrates its shard on
its own stream with grids small enough for all ranks' exchange kernels to be resident at once, and
the peer tables hold the other contexts' images (plain device pointers; across GPUs they are
NVLink-mapped symmetric memory).

Bars: after every exchanged launch every rank's image equals the element-wise sum of the images
the ranks' launches produce alone (bit-exact, integer); with binning only (n_steps = 0) that sum
equals the CPU oracle's histogram of the oracle's initial conditions, pixel for pixel; exchanging
contexts integrate bit-identically to plain ones; a missing peer ends in an error, not a hang.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402
from paper_1505_00344_b200.fireflies import ff_set_stream  # noqa: E402
from paper_1505_00344_b200._abi import FF_MAX_PEERS, FF_ERR_CUDA, FF_ERR_INVALID_ARG, FF_ERR_STATE, FFError  # noqa: E402

LZ_LO, LZ_HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]   # Fig. 3A box
LZ_P = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
GROUPS = [(20011, 2, 1, 0), (13007, 3, -1, 1)]           # (n, seed, direction, colour)


def make_rank(rank, world, image_shape, axes, view, grid_limit=16, stream=None):
    ctx = FF.Context(systems.lorenz(), [n for n, _, _, _ in GROUPS], rank=rank, world=world)
    if stream is not None:
        ff_set_stream(ctx.ctx, stream.cuda_stream)
        ctx.stream = stream
    for n, seed, d, colour in GROUPS:
        ctx.init_group(LZ_LO, LZ_HI, n, d, colour, seed)
    C_, H, W = image_shape
    img = torch.zeros((C_, H, W), dtype=torch.int32, device="cuda")
    ctx.project(axes, view, W, H, C_, image=img)
    ctx.set_grid_limit(grid_limit)
    return ctx, img


def exchanged_ranks(world, image_shape, axes, view, grid_limit=16, timeout_ms=20000.0):
    streams = [torch.cuda.Stream() for _ in range(world)]
    ranks = [make_rank(r, world, image_shape, axes, view, grid_limit, streams[r]) for r in range(world)]
    sigs = [torch.zeros(FF_MAX_PEERS, dtype=torch.int64, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    for r, (ctx, img) in enumerate(ranks):
        ctx.set_exchange(r, world, [i.data_ptr() for _, i in ranks], [s.data_ptr() for s in sigs], timeout_ms)
        ctx._keep_signals = sigs    # the signal words must outlive the contexts' exchanged launches
    return ranks, streams, sigs


def frame(ranks, streams, n_steps, dt=0.01):
    for (ctx, img), s in zip(ranks, streams):
        with torch.cuda.stream(s):
            img.zero_()
        ctx.step(n_steps, dt)
    for ctx, _ in ranks:
        ctx.sync()


def oracle_image(axes, view, W, H, C_):
    img = np.zeros((C_, H, W), np.uint32)
    for n, seed, _, colour in GROUPS:
        x = O.ic_uniform(LZ_LO, LZ_HI, seed, 0, n)
        O.histogram(x, axes, view, W, H, C_, colour, image=img)
    return img


@pytest.mark.parametrize("world", [1, 2, 3])
def test_bin_only_exchange_equals_oracle_histogram(world):
    """n_steps = 0: every rank's image after the exchange = the oracle's histogram of all
    particles' initial conditions (bit-exact), for a ragged image (C*H*W % 4 = 2)."""
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 29, 37)
    ranks, streams, _ = exchanged_ranks(world, shape, axes, view)
    frame(ranks, streams, 0)
    want = oracle_image(axes, view, shape[2], shape[1], shape[0])
    assert want.sum() > 0
    for _, img in ranks:
        assert np.array_equal(img.cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_exchange_equals_sum_of_rank_images_over_frames(world):
    """Lorenz, 3-D perspective image, several frames: exchanged images = sum of the images of plain
    (non-exchanging) replicas of the same shards, bit-exact; states bit-identical to the replicas."""
    M = views.look_at((0.0, -120.0, 25.0), (0.0, 0.0, 25.0), (0.0, 0.0, 1.0))
    P = views.perspective(45.0, 1.0, 1.0, 1000.0)
    mvp = (P @ M).astype(np.float32)
    axes, shape = [0, 1, 2], (2, 96, 128)
    ranks, streams, _ = exchanged_ranks(world, shape, axes, mvp)
    plain = [make_rank(r, world, shape, axes, mvp, grid_limit=0) for r in range(world)]
    for f in range(4):
        n = [3, 0, 25, 1][f]
        frame(ranks, streams, n)
        want = np.zeros(shape, np.uint64)
        for ctx, img in plain:
            img.zero_()
            ctx.step(n, 0.01)
            ctx.sync()
            want += img.cpu().numpy().view(np.uint32)
        assert want.sum() > 0
        for _, img in ranks:
            assert np.array_equal(img.cpu().numpy().view(np.uint32).astype(np.uint64), want), f"frame {f}"
    for (cx, _), (cp, _) in zip(ranks, plain):
        for g in range(len(GROUPS)):
            a, b = cx.read_state(g), cp.read_state(g)
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_exchange_accumulates_like_an_allreduce():
    """Without zeroing between frames the exchange sums the whole images (previous contents too),
    exactly as ff_step followed by an all-reduce would."""
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 32, 32)
    ranks, streams, _ = exchanged_ranks(2, shape, axes, view)
    frame(ranks, streams, 0)
    first = ranks[0][1].cpu().numpy().view(np.uint32).astype(np.uint64)
    for ctx, _ in ranks:        # no zeroing: each rank holds `first`, adds its own counts again
        ctx.step(0, 0.01)
    for ctx, _ in ranks:
        ctx.sync()
    got = ranks[1][1].cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(got, 2 * first + first)


def test_missing_peer_times_out_with_error_not_hang():
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 16, 16)
    ranks, streams, _ = exchanged_ranks(2, shape, axes, view, timeout_ms=300.0)
    ctx0, _ = ranks[0]
    ctx0.step(1, 0.01)                  # rank 1 never launches
    with pytest.raises(FFError) as e:
        ctx0.sync()
    assert e.value.status == FF_ERR_CUDA and "timed out" in str(e.value)
    ctx0.sync()                         # the flag is cleared; the context stays usable


def test_exchange_argument_errors():
    ctx = FF.Context(systems.lorenz(), [1000])
    ctx.init_group(LZ_LO, LZ_HI, 1000, 1, 0, 1)
    sig = torch.zeros(8, dtype=torch.int64, device="cuda")
    with pytest.raises(FFError) as e:
        ctx.set_exchange(0, 1, [sig.data_ptr()], [sig.data_ptr()])
    assert e.value.status == FF_ERR_STATE           # no image bound
    img = ctx.project([0, 1], [-20, 20, -30, 30], 16, 16, 1)
    other = torch.zeros_like(img)
    for args in [(0, 1, [other.data_ptr()], [sig.data_ptr()]),        # [rank] is not the bound image
                 (1, 1, [img.data_ptr()], [sig.data_ptr()]),          # rank >= world
                 (0, 9, [img.data_ptr()] * 9, [sig.data_ptr()] * 9),  # world > FF_MAX_PEERS
                 (0, 2, [img.data_ptr(), img.data_ptr() + 4], [sig.data_ptr()] * 2)]:  # misaligned
        with pytest.raises(FFError) as e:
            ctx.set_exchange(*args)
        assert e.value.status == FF_ERR_INVALID_ARG
    ctx.set_exchange(0, 1, [img.data_ptr()], [sig.data_ptr()])
    ctx.project([0, 1], [-20, 20, -30, 30], 16, 16, 1, image=other)   # rebinding ends the exchange
    ctx.step(1, 0.01)
    ctx.sync()
