"""GPU parity of the render post-process (NEXT row 3) -- bit-exact vs the oracle."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402


@pytest.mark.parametrize("radius", [0.5, 2.0, 3.7, 8.0])
def test_render_bit_exact(radius):
    n = 30000
    rng = np.random.default_rng(80)
    ctx = FF.Context(systems.lorenz(), [n, n])
    g0 = ctx.init_group([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], n, 1, 0, seed=2)
    g1 = ctx.init_group([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], n, -1, 1, seed=3)
    x0 = rng.normal(0, 6, (3, n)).astype(np.float32)
    x1 = rng.normal(0, 3, (3, n)).astype(np.float32)
    x0[0, :5000] = 0.5   # a dense column -> saturated pixels
    ctx.write_state(g0, x0)
    ctx.write_state(g1, x1)
    view = [-20.0, 20.0, -20.0, 20.0]
    ctx.project([0, 1], view, 200, 150, 2)
    colours = np.array([[0.0, 0.9, 0.2], [1.0, 0.4, 0.7]], np.float32)   # green / pink
    rgb = ctx.render(colours, 0.05, radius).cpu().numpy()
    img = O.histogram(x0, [0, 1], view, 200, 150, 2, 0)
    img = O.histogram(x1, [0, 1], view, 200, 150, 2, 1, image=img)
    want = O.render(img, colours, 0.05, radius)
    assert np.array_equal(rgb.view(np.uint32), want.view(np.uint32))
    assert rgb.max() == 1.0 and rgb.min() == 0.0


@pytest.mark.parametrize("ppt,tpb", [(2, 128), (4, 128), (1, 256)])
def test_position_colour_bit_exact(ppt, tpb):
    # colour linear in position: per-pixel colour sums and their render,
    # written through identical host state, bit-exact vs the oracle; includes a hot pixel (table path)
    n = 40000 + 1
    rng = np.random.default_rng(81)
    ctx = FF.Context(systems.lorenz(), [n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], n, 1, 0, seed=2)
    x = np.vstack([rng.normal(0, 8, n), rng.normal(0, 20, n), rng.uniform(0, 50, n)]).astype(np.float32)
    x[:, :8000] = np.array([[1.0], [2.0], [25.0]], np.float32)     # 8000 particles in one pixel
    ctx.write_state(g, x)
    M = views.lorenz_camera()
    img = ctx.project([0, 1, 2], M, 300, 300, 1)
    lo, hi = [-20.0, -30.0, 0.0], [20.0, 30.0, 50.0]
    col = ctx.project_colour(lo, hi)
    img.zero_()
    ctx.step(0, 0.01)   # bin-only launch (n = 0) with colour bound
    ctx.sync()
    want_c = O.colour_histogram(x, [0, 1, 2], M, 300, 300, lo, hi)
    assert np.array_equal(col.cpu().numpy().view(np.uint32), want_c)
    assert np.array_equal(ctx.read_image(), O.histogram(x, [0, 1, 2], M, 300, 300, 1, 0))
    rgb = ctx.render([[1, 1, 1]], 0.01, 2.0).cpu().numpy()
    assert np.array_equal(rgb.view(np.uint32), O.render_colour(want_c, 0.01, 2.0).view(np.uint32))


def test_render_after_fused_step_properties():
    # after a real fused launch: frame in [0, 1], lit exactly where the sprite footprint of a counted
    # pixel reaches (properties only -- the oracle never takes the GPU image as input)
    n = 1 << 16
    ctx = FF.Context(systems.lorenz(), [n])
    ctx.init_group([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], n, 1, 0, seed=2)
    img = ctx.project([0, 1, 2], views.lorenz_camera(), 512, 512, 1)
    img.zero_()
    ctx.step(200, 0.01)
    rgb = ctx.render([[1.0, 0.8, 0.0]], 0.2, 1.0).cpu().numpy()
    counts = ctx.read_image()[0]
    assert rgb.min() >= 0.0 and rgb.max() <= 1.0 and not rgb[2].any()
    assert np.array_equal(rgb[0] > 0, counts > 0)   # radius 1: only the centre tap has weight > 0
