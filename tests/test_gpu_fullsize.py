"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (default launch,
fused projection): sampled particles are recomputed one by one by the oracle from their own initial
conditions; the image is checked through properties that hold at any size."""
import numpy as np
import pytest

import oracle as O
from parity import dim_scales, finite_agreement, scaled_error

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402

LZ_LO, LZ_HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]


def sample(ctx, g, idx):
    return np.stack([ctx.read_state(g, int(i), 1)[:, 0] for i in idx], axis=1)


def oracle_at(lo, hi, seed, idx, model, p, h, steps, sweep_idx=-1, sv=None):
    x0 = np.hstack([O.ic_uniform(lo, hi, seed, int(i), 1) for i in idx])
    return O.rk4(model, x0, p, np.float32(h), steps, sweep_idx, sv)


def in_view_count_3d(x, M, W, H, margin=1e-3):
    """Particles whose perspective pixel lies inside the image, away from its border (float64 test
    logic with a margin) -- lower / upper bounds for the image sum."""
    X = np.vstack([x.astype(np.float64), np.ones((1, x.shape[1]))])
    c = M.astype(np.float64) @ X
    with np.errstate(all="ignore"):
        px, py = (c[0] / c[3] + 1) * W / 2, (c[1] / c[3] + 1) * H / 2
        ok = np.isfinite(px) & np.isfinite(py) & (c[3] > 0)
        inside = ok & (px >= margin) & (px < W - margin) & (py >= margin) & (py < H - margin)
        near = ok & ~inside & (px > -margin) & (px < W + margin) & (py > -margin) & (py < H + margin)
    return int(inside.sum()), int(near.sum())


def test_config2_lorenz_8M_fused_3d_image():
    n = 1 << 22
    ctx = FF.Context(systems.lorenz(), [n, n])
    gf = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=2)
    gb = ctx.init_group(LZ_LO, LZ_HI, n, -1, 1, seed=3)
    M = views.lorenz_camera()
    img = ctx.project([0, 1, 2], M, 1024, 1024, 2)
    img.zero_()
    ctx.step(30, 0.01)           # one fused launch, bench launch configuration
    p = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
    rng = np.random.default_rng(70)
    sc = dim_scales(LZ_LO, LZ_HI)
    for g, seed, h in ((gf, 2, 0.01), (gb, 3, -0.01)):
        idx = np.sort(rng.choice(n, 1500, replace=False))
        idx[-1] = n - 1
        got = sample(ctx, g, idx)
        want = oracle_at(LZ_LO, LZ_HI, seed, idx, O.LORENZ, p, h, 30)
        same, both = finite_agreement(got, want)
        assert same.all()
        e = scaled_error(got[:, both], want[:, both], sc).max(axis=0)
        if h > 0:
            assert e.max() <= 1e-5                          # Tier A (30 forward steps)
        else:
            assert np.percentile(e, 99) <= 1e-4 and e.max() <= 1e-2  # backward Tier B
    # image: every channel counts exactly the in-view particles of its group (up to border cases)
    im = ctx.read_image().astype(np.int64)
    for g, ch in ((gf, 0), (gb, 1)):
        inside, near = in_view_count_3d(ctx.group_view(g).cpu().numpy(), M, 1024, 1024)
        assert inside <= im[ch].sum() <= inside + near


def test_config4_sweep_16M_rho_y_image():
    n = 1 << 24
    ctx = FF.Context(systems.lorenz(), [n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=5)
    ctx.sweep_param(g, "r", 0.0, 200.0, 0, 5)
    view = [0.0, 200.0, -160.0, 160.0]
    img = ctx.project([3, 1], view, 2048, 1024, 1)
    img.zero_()
    ctx.step(10, 0.01)
    rng = np.random.default_rng(71)
    idx = np.sort(rng.choice(n, 1500, replace=False))
    sv = np.concatenate([O.sweep_values(0.0, 200.0, 0, 5, int(i), 1, n) for i in idx])
    got = sample(ctx, g, idx)
    want = oracle_at(LZ_LO, LZ_HI, 5, idx, O.LORENZ, np.array([10.0, 0.0, 8 / 3], np.float32), 0.01, 10, 1, sv)
    e = scaled_error(got, want, dim_scales(LZ_LO, LZ_HI)).max(axis=0)
    assert e.max() <= 1e-5                                   # Tier A (10 steps, swept r)
    im = ctx.read_image().astype(np.int64)
    y = ctx.group_view(g)[1].cpu().numpy()
    inside = int(((y >= -160) & (y < 160)).sum())           # r is always inside [0, 200)
    assert im.sum() == inside
    # the r columns: r is uniform in [0, 200), and for r < 50 every particle is still inside the y
    # window after 10 steps, so each of the first 512 columns holds ~n/2048 particles
    col = im[0].sum(axis=0)[:512]
    assert abs(col.mean() - n / 2048) < 20 and col.min() > 0.9 * n / 2048


def test_next4_stn_bifurcation_8M_reset_3d_image():
    """NEXT row 4 at the bench's size and launch (`bench.py --config stn_bif3d`): 2^22 forward + 2^22
    backward STN-GPe particles, w_ss swept over [0, 12), reset to the unit square, one fused launch
    of 100 steps + reset + 3-D binning of (x, y, w_ss) -- the pipe-balanced kernel. Sampled particles
    the oracle does not reset: Tier A; their reset decision agrees; every channel counts exactly
    the in-view particles of its group (up to border cases)."""
    s = systems.stn_gpe()
    p = np.array([q[1] for q in s.params], np.float32)
    n = 1 << 22
    ctx = FF.Context(s, [n, n])
    gf = ctx.init_group([0.0, 0.0], [1.0, 1.0], n, 1, 0, seed=21)
    gb = ctx.init_group([0.0, 0.0], [1.0, 1.0], n, -1, 1, seed=22)
    for g in (gf, gb):
        ctx.sweep_param(g, "w_ss", 0.0, 12.0, 0, 23)
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)
    M = views.box_camera([0.0, 0.0, 0.0], [1.0, 1.0, 12.0])
    img = ctx.project([0, 1, 2], M, 1024, 1024, 2)
    img.zero_()
    ctx.step(100, 0.01)
    rng = np.random.default_rng(72)
    sv_all = O.sweep_values(0.0, 12.0, 0, 23, 0, n, n)
    im = ctx.read_image().astype(np.int64)
    for g, seed, h, ch in ((gf, 21, 0.01, 0), (gb, 22, -0.01, 1)):
        idx = np.sort(rng.choice(n, 1500, replace=False))
        idx[-1] = n - 1
        sv = sv_all[idx]
        want = oracle_at([0.0, 0.0], [1.0, 1.0], seed, idx, O.STN, p, h, 100, 0, sv)
        got = sample(ctx, g, idx)
        ep = np.array([ctx.read_epochs(g, int(i), 1)[0] for i in idx])
        kept = np.all(np.isfinite(want) & (want >= 0.0) & (want <= 1.0), axis=0)
        assert np.count_nonzero((ep == 0) != kept) <= 3
        both = kept & (ep == 0)
        assert both.sum() > 100
        assert scaled_error(got[:, both], want[:, both], [1.0, 1.0]).max() <= 1e-5
        x = ctx.group_view(g).cpu().numpy()
        assert np.all((x >= 0.0) & (x <= 1.0))             # after the reset every particle is in the box
        inside, near = in_view_count_3d(np.vstack([x, sv_all[None, :]]), M, 1024, 1024)
        assert inside <= im[ch].sum() <= inside + near


def test_config3_hh_1M():
    s = systems.hh_ring(3)
    d = {p[0]: p[1] for p in s.params}
    p = np.array([d[k] for k in O.hh_param_names(3)], np.float32)
    lo, hi = [-20.0, 0, 0, 0, 0] * 3, [100.0, 1, 1, 1, 1] * 3
    n = 1 << 20
    ctx = FF.Context(s, [n])
    g = ctx.init_group(lo, hi, n, 1, 0, seed=4)
    img = ctx.project([0, 5], [-20.0, 120.0, -20.0, 120.0], 1024, 1024, 1)
    img.zero_()
    ctx.step(10, 0.01)
    rng = np.random.default_rng(72)
    idx = np.sort(rng.choice(n, 400, replace=False))
    got = sample(ctx, g, idx)
    want = oracle_at(lo, hi, 4, idx, O.HH, p, 0.01, 10)
    assert scaled_error(got, want, dim_scales(lo, hi)).max() <= 1e-5
    x = ctx.group_view(g).cpu().numpy()
    inside = int(((x[0] >= -20) & (x[0] < 120) & (x[5] >= -20) & (x[5] < 120)).sum())
    assert int(ctx.read_image().sum()) == inside


@pytest.mark.slow
def test_config5_lorenz_1B_one_gpu():
    # configs[4] at its full 2^30 particles on one B200 (12 GB of state); 5 fused steps.
    n = 1 << 30
    ctx = FF.Context(systems.lorenz(), [n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=6)
    M = views.lorenz_camera()
    img = ctx.project([0, 1, 2], M, 1024, 1024, 1)
    img.zero_()
    ctx.step(5, 0.01)
    p = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
    idx = np.array([0, 1, 12345, n // 2, n - 2, n - 1], np.int64)
    got = sample(ctx, g, idx)
    want = oracle_at(LZ_LO, LZ_HI, 6, idx, O.LORENZ, p, 0.01, 5)
    assert scaled_error(got, want, dim_scales(LZ_LO, LZ_HI)).max() <= 1e-5
    assert 0 < int(ctx.read_image().astype(np.int64).sum()) <= n
