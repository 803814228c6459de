"""CUDA-graph capture of frames (the main loop of PAPER.md:242 replays the same frame):
a captured frame (image zero + fused step with the reset rule) replayed k times equals k ordinary
frames of a twin context bit for bit -- state, epochs and image -- and ordinary launches after the
replays still agree (the tile counter restarts per launch once a context was captured). Capture
restrictions fail loudly."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402
from paper_1505_00344_b200._abi import FFError, FF_ERR_STATE  # noqa: E402

LO, HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]


def make(n):
    ctx = FF.Context(systems.lorenz(), [n, n])
    gf = ctx.init_group(LO, HI, n, 1, 0, seed=2)
    gb = ctx.init_group(LO, HI, n, -1, 1, seed=3)
    ctx.set_reset(True)
    img = ctx.project([0, 1, 2], views.lorenz_camera(), 256, 192, 2)
    return ctx, (gf, gb), img


@pytest.mark.parametrize("S", [1, 10, 100])
def test_replayed_frames_equal_ordinary_frames(S):
    n = 200000 + 17
    a, ga, ia = make(n)
    b, gb, ib = make(n)

    def frame():
        ia.zero_()
        a.step(S, 0.01)
    frame()                      # compiles the kernel outside the capture
    ib.zero_()
    b.step(S, 0.01)
    g = a.capture(frame)
    for _ in range(4):
        g.replay()
        ib.zero_()
        b.step(S, 0.01)
    a.step(S, 0.01)              # an ordinary launch after the replays, accumulating
    b.step(S, 0.01)
    torch.cuda.synchronize()
    for x, y in zip(ga, gb):
        assert np.array_equal(a.read_state(x).view(np.uint32), b.read_state(y).view(np.uint32))
        assert np.array_equal(a.read_epochs(x), b.read_epochs(y))
    assert np.array_equal(a.read_image(), b.read_image()) and int(a.read_image().sum()) > 0
    if S >= 10:   # (6 steps are too few for a backward particle to blow up)
        assert a.read_epochs(ga[1]).sum() > 0    # the backward group was reset inside the replays


def test_capture_restrictions():
    a, ga, ia = make(5000)
    a.set_reset(True, None, None, 5.0)            # age rule: needs each launch's time
    a.step(10, 0.01)
    with pytest.raises(FFError) as e:
        a.capture(lambda: a.step(10, 0.01))
    assert e.value.status == FF_ERR_STATE
    a.set_reset(True)
    a.set_launch(1, 512)                          # a kernel variant never launched: not compiled yet
    with pytest.raises(FFError) as e:
        a.capture(lambda: a.step(1, 0.01))
    assert e.value.status == FF_ERR_STATE
