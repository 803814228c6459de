"""GPU tests of the fused (push) image exchange (ff_set_exchange_push; SURVEY.md 8(e) "Fused option",
8(f) NEXT 2): the histogram's own reductions go to every rank's image -- red.add over peer memory here
(on one GPU the ranks are contexts sharing it, their images the peers'), multimem.red through an NVLS
multicast address on a multicast-capable system (same kernels apart from that one instruction,
tests/test_gpu_exchange_nvls.py) -- between a barrier before and a barrier after each launch.

Bars: with every rank's image zeroed per frame, every rank's image after each frame equals the sum of
the images plain (non-exchanging) replicas of the same shards produce (bit-exact, integer), and with
binning only the oracle's histogram of all particles' initial conditions, pixel for pixel; in every
launch variant and histogram regime (dispersed, one-pixel warps, block hash table and its overflow);
states bit-identical to the replicas; without zeroing the launches accumulate like the unsharded run
(not like the sum pass's all-reduce); a missing peer ends in an error, not a hang.
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
from paper_1505_00344_b200._abi import FF_ERR_CUDA, FF_ERR_INVALID_ARG, FF_ERR_STATE, FFError, check, lib  # noqa: E402
from test_gpu_exchange import GROUPS, LZ_HI, LZ_LO, exchanged_ranks, frame, make_rank, oracle_image  # noqa: E402


def pushing_ranks(world, shape, axes, view, launch=None, timeout_ms=20000.0):
    ranks, streams, sigs = exchanged_ranks(world, shape, axes, view, timeout_ms=timeout_ms)
    for ctx, _ in ranks:
        if launch:
            ctx.set_launch(*launch)
        ctx.set_exchange_push(True)
    return ranks, streams, sigs


def mvp():
    M = views.look_at((0.0, -120.0, 25.0), (0.0, 0.0, 25.0), (0.0, 0.0, 1.0))
    P = views.perspective(45.0, 1.0, 1.0, 1000.0)
    return (P @ M).astype(np.float32)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_bin_only_push_equals_oracle_histogram(world):
    """n_steps = 0: every rank's image = the oracle's histogram of all particles' initial conditions
    (bit-exact), ragged image (C*H*W % 4 = 2)."""
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 29, 37)
    ranks, streams, _ = pushing_ranks(world, shape, axes, view)
    frame(ranks, streams, 0)
    want = oracle_image(axes, view, shape[2], shape[1], shape[0])
    assert want.sum() > 0
    for _, img in ranks:
        assert np.array_equal(img.cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("launch", [None, (4, 128), (2, 128), (2, 256), (1, 128), (1, 512)])
@pytest.mark.parametrize("world", [2, 4])
def test_push_equals_sum_of_rank_images_over_frames(world, launch):
    """Lorenz, 3-D perspective image, frames of 3, 0, 25, 1 and 100 steps, in every step-kernel
    variant: each rank's image = the sum of plain replicas' images, bit-exact; states identical."""
    axes, shape, M = [0, 1, 2], (2, 96, 128), mvp()
    ranks, streams, _ = pushing_ranks(world, shape, axes, M, launch)
    plain = [make_rank(r, world, shape, axes, M, grid_limit=0) for r in range(world)]
    for f, n in enumerate([3, 0, 25, 1, 100]):
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
            assert np.array_equal(cx.read_state(g).view(np.uint32), cp.read_state(g).view(np.uint32))


@pytest.mark.parametrize("shape", [(2, 1, 1), (2, 2, 3), (2, 40, 40)])
def test_push_concentrated_regimes(shape):
    """Images of 1, 6 and 1600 pixels per channel: whole warps in one pixel, the block hash table
    (flushed at block exit through the push reductions), and a crowded table's direct reductions.
    Bin-only frame against the oracle, then an integrating frame against plain replicas."""
    axes, view = [0, 2], [-20.0, 20.0, 0.0, 50.0]
    world = 3
    ranks, streams, _ = pushing_ranks(world, shape, axes, view)
    frame(ranks, streams, 0)
    want = oracle_image(axes, view, shape[2], shape[1], shape[0])
    for _, img in ranks:
        assert np.array_equal(img.cpu().numpy().view(np.uint32), want)
    plain = [make_rank(r, world, shape, axes, view, grid_limit=0) for r in range(world)]
    frame(ranks, streams, 10)
    want = np.zeros(shape, np.uint64)
    for ctx, img in plain:
        img.zero_()
        ctx.step(10, 0.01)
        ctx.sync()
        want += img.cpu().numpy().view(np.uint32)
    for _, img in ranks:
        assert np.array_equal(img.cpu().numpy().view(np.uint32).astype(np.uint64), want)


def test_push_accumulates_like_the_unsharded_run():
    """Without zeroing, a pushing launch adds the ranks' total counts to every image (previous
    contents kept, not summed over ranks): two bin-only launches give 2x the histogram -- the
    unsharded run's image -- where the sum pass gives 3x (tests/test_gpu_exchange.py)."""
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 32, 32)
    ranks, streams, _ = pushing_ranks(2, shape, axes, view)
    frame(ranks, streams, 0)
    first = ranks[0][1].cpu().numpy().view(np.uint32).astype(np.uint64)
    for ctx, _ in ranks:
        ctx.step(0, 0.01)
    for ctx, _ in ranks:
        ctx.sync()
    for _, img in ranks:
        assert np.array_equal(img.cpu().numpy().view(np.uint32).astype(np.uint64), 2 * first)
    single = make_rank(0, 1, shape, axes, view, grid_limit=0)[0]
    single.step(0, 0.01)
    assert np.array_equal(single.read_image().astype(np.uint64), 2 * first)


@pytest.mark.parametrize("sizes", [[(20011, 2, 1, 0), (13007, 3, -1, 1)], [(2, 2, 1, 0), (1, 3, -1, 1)]])
def test_push_with_reset_rule_and_empty_rank(sizes):
    """The bench's frame (non-finite reset, forward + backward Lorenz) over 3 ranks; with groups of 2
    and 1 particles rank 0 owns none (it contributes nothing but still takes part in both barriers of
    every launch) and every rank's image must still be the unsharded image."""
    from paper_1505_00344_b200.fireflies import ff_set_stream
    axes, shape, M = [0, 1, 2], (2, 64, 64), mvp()
    world = 3
    streams = [torch.cuda.Stream() for _ in range(world)]
    ranks = []
    for r in range(world):
        ctx = FF.Context(systems.lorenz(), [n for n, _, _, _ in sizes], rank=r, world=world)
        ff_set_stream(ctx.ctx, streams[r].cuda_stream)
        ctx.stream = streams[r]
        for n, seed, d, colour in sizes:
            ctx.init_group(LZ_LO, LZ_HI, n, d, colour, seed)
        ctx.set_reset(True, None, None, 0.0)
        img = torch.zeros(shape, dtype=torch.int32, device="cuda")
        ctx.project(axes, M, shape[2], shape[1], shape[0], image=img)
        ctx.set_grid_limit(16)
        ranks.append((ctx, img))
    sigs = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    for r, (ctx, _) in enumerate(ranks):
        ctx.set_exchange(r, world, [i.data_ptr() for _, i in ranks], [s.data_ptr() for s in sigs], 20000.0)
        ctx.set_exchange_push(True)
        ctx._keep_signals = sigs
    single = FF.Context(systems.lorenz(), [n for n, _, _, _ in sizes])
    for n, seed, d, colour in sizes:
        single.init_group(LZ_LO, LZ_HI, n, d, colour, seed)
    single.set_reset(True, None, None, 0.0)
    simg = single.project(axes, M, shape[2], shape[1], shape[0])
    for n in (100, 100, 50):
        frame(ranks, streams, n)
        simg.zero_()
        single.step(n, 0.01)
        want = single.read_image()
        assert want.sum() > 0 or sizes[0][0] < 100
        for _, img in ranks:
            assert np.array_equal(img.cpu().numpy().view(np.uint32), want)


def test_push_missing_peer_times_out_with_error_not_hang():
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 16, 16)
    ranks, streams, _ = pushing_ranks(2, shape, axes, view, timeout_ms=300.0)
    ctx0, _ = ranks[0]
    ctx0.step(1, 0.01)                  # rank 1 never launches
    with pytest.raises(FFError) as e:
        ctx0.sync()
    assert e.value.status == FF_ERR_CUDA and "timed out" in str(e.value)
    ctx0.sync()                         # the flag is cleared; the context stays usable


def test_push_off_returns_to_the_sum_pass_and_argument_errors():
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 32, 32)
    ranks, streams, _ = pushing_ranks(2, shape, axes, view)
    frame(ranks, streams, 0)
    first = ranks[0][1].cpu().numpy().view(np.uint32).astype(np.uint64)
    for ctx, _ in ranks:
        ctx.set_exchange_push(False)
    for ctx, _ in ranks:                # sum pass again: previous contents summed over ranks
        ctx.step(0, 0.01)
    for ctx, _ in ranks:
        ctx.sync()
    assert np.array_equal(ranks[1][1].cpu().numpy().view(np.uint32).astype(np.uint64), 3 * first)
    ctx = ranks[0][0]
    with pytest.raises(FFError) as e:
        check(lib().ff_set_exchange_push(ctx.ctx, 2, None))   # on must be 0 or 1
    assert e.value.status == FF_ERR_INVALID_ARG
    with pytest.raises(FFError) as e:
        ctx.set_exchange_push(True, 8)  # misaligned multicast address
    assert e.value.status == FF_ERR_INVALID_ARG
    lone = FF.Context(systems.lorenz(), [1000])
    lone.init_group(LZ_LO, LZ_HI, 1000, 1, 0, 1)
    with pytest.raises(FFError) as e:
        lone.set_exchange_push(True)    # no exchange set
    assert e.value.status == FF_ERR_STATE


@pytest.mark.parametrize("push", [False, True])
def test_exchange_full_size_bench_launch(push):
    """configs[1] at full size in the bench's launch (2^22 forward + 2^22 backward Lorenz particles, the
    non-finite reset rule, 3-D 1024^2 x 2 image, S = 100 and S = 1 frames, default kernel choice and
    full grids) sharded over two ranks as contexts on one GPU: after each frame both ranks' images
    equal the unsharded run's image bit for bit, for the sum-pass exchange and for the push exchange."""
    from paper_1505_00344_b200.fireflies import ff_set_stream
    n = 1 << 22
    sizes = [(n, 2, 1, 0), (n, 3, -1, 1)]
    axes, shape, M = [0, 1, 2], (2, 1024, 1024), views.lorenz_camera()
    world = 2
    streams = [torch.cuda.Stream() for _ in range(world)]
    ranks = []
    for r in range(world):
        ctx = FF.Context(systems.lorenz(), [k for k, _, _, _ in sizes], rank=r, world=world)
        ff_set_stream(ctx.ctx, streams[r].cuda_stream)
        ctx.stream = streams[r]
        for k, seed, d, colour in sizes:
            ctx.init_group(LZ_LO, LZ_HI, k, d, colour, seed)
        ctx.set_reset(True, None, None, 0.0)
        img = torch.zeros(shape, dtype=torch.int32, device="cuda")
        ctx.project(axes, M, shape[2], shape[1], shape[0], image=img)
        ranks.append((ctx, img))
    sigs = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    for r, (ctx, _) in enumerate(ranks):
        ctx.set_exchange(r, world, [i.data_ptr() for _, i in ranks], [s.data_ptr() for s in sigs], 20000.0)
        if push:
            ctx.set_exchange_push(True)
        ctx._keep_signals = sigs
    single = FF.Context(systems.lorenz(), [k for k, _, _, _ in sizes])
    for k, seed, d, colour in sizes:
        single.init_group(LZ_LO, LZ_HI, k, d, colour, seed)
    single.set_reset(True, None, None, 0.0)
    simg = single.project(axes, M, shape[2], shape[1], shape[0])
    for S in (100, 1, 100):
        frame(ranks, streams, S)
        simg.zero_()
        single.step(S, 0.01)
        want = single.read_image()
        assert want.sum() > (1 << 22)          # both groups binned (the reset keeps the backward one in view)
        for _, img in ranks:
            assert np.array_equal(img.cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("push", [False, True])
def test_exchanging_contexts_refuse_graph_capture(push):
    """A captured frame would replay barrier values of the capture forever, so an exchanging context
    (sum pass or push) refuses CUDA-graph capture with FF_ERR_STATE and stays usable afterwards."""
    axes, view, shape = [0, 2], [-20.0, 20.0, 0.0, 50.0], (2, 16, 16)
    ranks, streams, _ = (pushing_ranks if push else exchanged_ranks)(2, shape, axes, view)
    frame(ranks, streams, 1)
    ctx = ranks[0][0]
    with pytest.raises(FFError) as e:
        ctx.capture(lambda: ctx.step(1, 0.01))
    assert e.value.status == FF_ERR_STATE
    frame(ranks, streams, 1)                       # both ranks still exchange normally
    want = np.zeros(shape, np.uint64)
    for r in range(2):
        c, im = make_rank(r, 2, shape, axes, view, grid_limit=0)
        c.step(2, 0.01)
        im.zero_()
        c.step(0, 0.01)
        c.sync()
        want += im.cpu().numpy().view(np.uint32)
    for _, img in ranks:
        assert np.array_equal(img.cpu().numpy().view(np.uint32).astype(np.uint64), want)
