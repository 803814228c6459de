"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Bars: initial conditions and swept values bit-exact; histograms bit-exact on
identical coordinates; state within the scaled tolerance e <= 1e-5 (Tier A) over the horizons
calibrated in SURVEY.md 8(c), statistical Tier B beyond them.
"""
import numpy as np
import pytest

import oracle as O
from parity import dim_scales, finite_agreement, oracle_group, scaled_error, tier_a

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402
from paper_1505_00344_b200._abi import FFError, FF_ERR_RANGE, FF_ERR_STATE, FF_ERR_UNKNOWN_SYMBOL  # noqa: E402

LZ_LO, LZ_HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]   # Fig. 3A box
LZ_P = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
LAUNCHES = [(1, 128), (1, 256), (1, 512), (2, 128), (2, 256), (4, 128)]


def lorenz_ctx(sizes, r=28.0):
    ctx = FF.Context(systems.lorenz(), sizes)
    ctx.set_param("r", r)
    return ctx


# ----------------------------------------------------------------------------- initial conditions
def test_ic_bit_exact_and_padding_nan():
    sizes = [5000, 3001, 1]
    ctx = lorenz_ctx(sizes)
    gs = [ctx.init_group(LZ_LO, LZ_HI, n, 1 if k != 1 else -1, 0, seed=2 + k) for k, n in enumerate(sizes)]
    for k, (g, n) in enumerate(zip(gs, sizes)):
        got = ctx.read_state(g)
        want = O.ic_uniform(LZ_LO, LZ_HI, 2 + k, 0, n)
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        s, nl, _ = ctx.group_info(g)
        pad = ctx.state[:, s + nl:s + ((nl + 511) // 512) * 512].cpu().numpy()
        assert np.all(np.isnan(pad))


def test_ic_golden_values():
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ic_golden.json")))
    ctx = lorenz_ctx([4194305])
    g = ctx.init_group(LZ_LO, LZ_HI, 4194305, 1, 0, seed=2)
    for c in gold["ic"]:
        x = ctx.read_state(g, c["index"], 1)[:, 0]
        assert [int(b) for b in x.view(np.uint32)] == [int(b, 16) for b in c["bits"]]


# ----------------------------------------------------------------------------- integrator parity
@pytest.mark.parametrize("ppt,tpb", LAUNCHES)
def test_lorenz_r28_tier_a(ppt, tpb):
    # Tier A horizons: forward 30 steps, backward 10 steps -- set by the oracle-only proxy (FP32 vs
    # FP64 oracle from the same ICs, tools/calibrate_tiers.py -> profiles/r02_tier_calibration.json:
    # forward max 1.4e-6 at 30 steps; backward 8.9e-7 at 10 but 1.2e-5 at 20 steps -- backward Lorenz
    # particles blow up, so rounding differences grow fast), not by the GPU itself.
    n = 20000 + 77  # several tiles and a ragged tail
    ctx = lorenz_ctx([n, n])
    ctx.set_launch(ppt, tpb)
    gf = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=2)
    gb = ctx.init_group(LZ_LO, LZ_HI, n, -1, 1, seed=3)
    sc = dim_scales(LZ_LO, LZ_HI)
    ctx.step(4, 0.01)
    ctx.step(6, 0.01)
    want_b = oracle_group(O.LORENZ, LZ_LO, LZ_HI, 3, 0, n, LZ_P, -0.01, 10)
    assert tier_a(ctx.read_state(gb), want_b, sc) <= 1e-5
    ctx.step(20, 0.01)
    want_f = oracle_group(O.LORENZ, LZ_LO, LZ_HI, 2, 0, n, LZ_P, 0.01, 30)
    assert tier_a(ctx.read_state(gf), want_f, sc) <= 1e-5
    # backward group at 30 steps: Tier B (measured p99 1.6e-5, max 3.4e-4 over 1e5 particles)
    want_b = O.rk4(O.LORENZ, want_b, LZ_P, np.float32(-0.01), 20)
    got = ctx.read_state(gb)
    same, both = finite_agreement(got, want_b)
    assert same.all()
    e = scaled_error(got[:, both], want_b[:, both], sc).max(axis=0)
    assert np.percentile(e, 99) <= 1e-4 and e.max() <= 1e-2


def test_lorenz_r28_tier_b_100_steps():
    n = 50000
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=2)
    ctx.step(100, 0.01)
    want = oracle_group(O.LORENZ, LZ_LO, LZ_HI, 2, 0, n, LZ_P, 0.01, 100)
    got = ctx.read_state(g)
    e = scaled_error(got, want, dim_scales(LZ_LO, LZ_HI)).max(axis=0)
    assert np.percentile(e, 99) <= 1e-5 and np.percentile(e, 99.99) <= 1e-3


def test_lorenz_r05_tier_a_1000_steps_and_origin_fixed():
    n = 10000
    ctx = lorenz_ctx([n, 512], r=0.5)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=5)
    g0 = ctx.init_group([0.0, 0.0, 0.0], [1e-30, 1e-30, 1e-30], 512, 1, 0, seed=6)
    ctx.write_state(g0, np.zeros((3, 512), np.float32))
    ctx.step(1000, 0.01)
    p = np.array([10.0, 0.5, 8.0 / 3.0], np.float32)
    want = oracle_group(O.LORENZ, LZ_LO, LZ_HI, 5, 0, n, p, 0.01, 1000)
    assert tier_a(ctx.read_state(g), want, dim_scales(LZ_LO, LZ_HI)) <= 1e-5
    assert np.all(ctx.read_state(g0) == 0)   # PAPER.md:87 fixed point, bit-exact


def test_linear_closed_form_on_gpu():
    # x' = -x, h = 0.1: one RK4 step is T4(-0.1) = 0.9048375, h = -0.1 -> 1.1051708
    ctx = FF.Context(systems.linear([[-1.0]]), [512, 512])
    g1 = ctx.init_group([1.0], [1.0000001], 512, 1, 0, 1)
    g2 = ctx.init_group([1.0], [1.0000001], 512, -1, 0, 1)
    ctx.write_state(g1, np.ones((1, 512), np.float32))
    ctx.write_state(g2, np.ones((1, 512), np.float32))
    ctx.step(1, 0.1)
    assert np.allclose(ctx.read_state(g1), 0.9048375, rtol=2e-7, atol=0)
    assert np.allclose(ctx.read_state(g2), 1.1051708333, rtol=2e-7, atol=0)


def test_zero_steps_is_identity_and_params_take_effect():
    n = 4096
    ctx = lorenz_ctx([n], r=0.5)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=9)
    x0 = ctx.read_state(g)
    ctx.step(0, 0.01)
    assert np.array_equal(ctx.read_state(g), x0)
    ctx.step(20, 0.01)
    ctx.set_param("r", 28.0)  # the next launch sees the new value
    ctx.step(10, 0.01)
    want = O.rk4(O.LORENZ, x0, np.array([10, 0.5, 8 / 3], np.float32), np.float32(0.01), 20)
    want = O.rk4(O.LORENZ, want, LZ_P, np.float32(0.01), 10)
    assert tier_a(ctx.read_state(g), want, dim_scales(LZ_LO, LZ_HI)) <= 1e-5


def test_uniform_factors_follow_param_changes():
    """sigma (Lorenz dx/dt = sigma (y - x)) and 1/tau (STN-GPe) are factored out of the generated RHS
    into step constants the host computes per launch: a parameter change between
    launches takes effect exactly like any other."""
    n = 8192 + 3
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=12)
    x0 = ctx.read_state(g)
    ctx.step(10, 0.01)
    ctx.set_param("sigma", 14.0)
    ctx.step(10, 0.01)
    want = O.rk4(O.LORENZ, x0, LZ_P, np.float32(0.01), 10)
    want = O.rk4(O.LORENZ, want, np.array([14.0, 28.0, 8.0 / 3.0], np.float32), np.float32(0.01), 10)
    assert tier_a(ctx.read_state(g), want, dim_scales(LZ_LO, LZ_HI)) <= 1e-5

    p, sdef = stn_params()
    ctx = FF.Context(sdef, [n])
    g = ctx.init_group([0.0, 0.0], [1.0, 1.0], n, 1, 0, seed=13)
    x0 = ctx.read_state(g)
    ctx.step(50, 0.01)
    names = [q[0] for q in sdef.params]
    ctx.set_param("tau_s", 2.5)
    ctx.set_param("tau_g", 0.7)
    ctx.step(50, 0.01)
    p2 = p.copy()
    p2[names.index("tau_s")], p2[names.index("tau_g")] = 2.5, 0.7
    want = O.rk4(O.STN, x0, p, np.float32(0.01), 50)
    want = O.rk4(O.STN, want, p2, np.float32(0.01), 50)
    assert tier_a(ctx.read_state(g), want, [1.0, 1.0]) <= 1e-5


@pytest.mark.parametrize("mode", [0, 1])
def test_swept_factor_stays_per_particle(mode):
    """Sweeping the factored parameter itself (sigma): it is per particle then, so it is not
    factored out; the result still matches the oracle's per-particle sigma."""
    n = 20000 + 9
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=14)
    ctx.sweep_param(g, "sigma", 5.0, 15.0, mode, seed=15)
    sv = O.sweep_values(5.0, 15.0, mode, 15, 0, n, n)
    ctx.step(10, 0.01)
    xo = O.rk4(O.LORENZ, O.ic_uniform(LZ_LO, LZ_HI, 14, 0, n), LZ_P, np.float32(0.01), 10, 0, sv)
    assert tier_a(ctx.read_state(g), xo, dim_scales(LZ_LO, LZ_HI)) <= 1e-5


def stn_params():
    s = systems.stn_gpe()
    return np.array([p[1] for p in s.params], np.float32), s


def test_stn_forward_1000_backward_100():
    # Config 1 shape (BASELINE.json configs[0]): 5k forward + 5k backward, dt = 0.01.
    p, s = stn_params()
    ctx = FF.Context(s, [5000, 5000])
    gf = ctx.init_group([0, 0], [1, 1], 5000, 1, 0, seed=1)
    gb = ctx.init_group([0, 0], [1, 1], 5000, -1, 1, seed=11)
    ctx.step(100, 0.01)
    wb = oracle_group(O.STN, [0, 0], [1, 1], 11, 0, 5000, p, -0.01, 100)
    assert tier_a(ctx.read_state(gb), wb, [1.0, 1.0]) <= 1e-5
    ctx.step(900, 0.01)
    wf = oracle_group(O.STN, [0, 0], [1, 1], 1, 0, 5000, p, 0.01, 1000)
    assert tier_a(ctx.read_state(gf), wf, [1.0, 1.0]) <= 1e-5


def test_stn_backward_group_1000_steps_tier_b():
    """configs[0]'s backward group over its full 1000 steps (SURVEY.md 8(c) Tier B: p99 <= 1e-4, max
    <= 1e-2; the oracle-only proxy FP32 vs FP64 gives p99 1.6e-5, max 2.9e-3,
    profiles/r02_tier_calibration.json), finite on both sides or on neither."""
    p, s = stn_params()
    ctx = FF.Context(s, [5000, 5000])
    ctx.init_group([0, 0], [1, 1], 5000, 1, 0, seed=1)
    gb = ctx.init_group([0, 0], [1, 1], 5000, -1, 1, seed=11)
    ctx.step(1000, 0.01)
    want = oracle_group(O.STN, [0, 0], [1, 1], 11, 0, 5000, p, -0.01, 1000)
    got = ctx.read_state(gb)
    same, both = finite_agreement(got, want)
    assert same.all()
    e = scaled_error(got[:, both], want[:, both], [1.0, 1.0]).max(axis=0)
    assert np.percentile(e, 99) <= 1e-4 and e.max() <= 1e-2


def test_stn_limit_cycle_tier_b():
    p, s = stn_params()
    p[0] = 7.8
    ctx = FF.Context(s, [4000])
    ctx.set_param("w_ss", 7.8)
    g = ctx.init_group([0, 0], [1, 1], 4000, 1, 0, seed=3)
    ctx.step(1000, 0.01)
    want = oracle_group(O.STN, [0, 0], [1, 1], 3, 0, 4000, p, 0.01, 1000)
    e = scaled_error(ctx.read_state(g), want, [1.0, 1.0]).max(axis=0)
    assert np.percentile(e, 99) <= 1e-4 and e.max() <= 1e-3


HH_LO = [-20.0, 0, 0, 0, 0] * 3
HH_HI = [100.0, 1, 1, 1, 1] * 3


def hh_params(s):
    names = O.hh_param_names(3)
    d = {p[0]: p[1] for p in s.params}
    return np.array([d[k] for k in names], np.float32)


@pytest.mark.parametrize("ppt", [1, 2])
def test_hh_ring_tier_a_10_steps_tier_b_100(ppt):
    s = systems.hh_ring(3)
    p = hh_params(s)
    n = 6000
    ctx = FF.Context(s, [n])
    ctx.set_launch(ppt, 256 if ppt == 1 else 128)
    g = ctx.init_group(HH_LO, HH_HI, n, 1, 0, seed=4)
    sc = dim_scales(HH_LO, HH_HI)
    ctx.step(10, 0.01)
    want = oracle_group(O.HH, HH_LO, HH_HI, 4, 0, n, p, 0.01, 10)
    assert tier_a(ctx.read_state(g), want, sc) <= 1e-5
    ctx.step(90, 0.01)
    want = O.rk4(O.HH, want, p, np.float32(0.01), 90)
    got = ctx.read_state(g)
    same, both = finite_agreement(got, want)
    assert same.all()
    e = scaled_error(got[:, both], want[:, both], sc).max(axis=0)
    assert np.percentile(e, 99) <= 1e-5 and e.max() <= 1e-3


# ----------------------------------------------------------------------------- sweep
@pytest.mark.parametrize("mode", [0, 1])
def test_sweep_values_bit_exact_and_parity(mode):
    n = 30000 + 5
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=5)
    ctx.sweep_param(g, "r", 0.0, 200.0, mode, seed=5)
    # the swept value is axis `dim` (= 3); a (r, r) window image pins every value bit-exactly
    sv = O.sweep_values(0.0, 200.0, mode, 5, 0, n, n)
    W = 4096
    img = ctx.project([3, 3], [0.0, 200.0, 0.0, 200.0], W, 1, 1)
    want = O.histogram(np.zeros((3, n), np.float32), [3, 3], [0.0, 200.0, 0.0, 200.0], W, 1, 1, 0, sweep_vals=sv)
    assert np.array_equal(ctx.read_image(), want)
    ctx.step(10, 0.01)
    xo = O.rk4(O.LORENZ, O.ic_uniform(LZ_LO, LZ_HI, 5, 0, n), LZ_P, np.float32(0.01), 10, 1, sv)
    assert tier_a(ctx.read_state(g), xo, dim_scales(LZ_LO, LZ_HI)) <= 1e-5
    # lifted parameter unchanged: rebinning the swept axis after stepping gives the same image
    img.zero_()
    ctx.project([3, 3], [0.0, 200.0, 0.0, 200.0], W, 1, 1, image=img)
    assert np.array_equal(ctx.read_image(), want)


def test_sweep_and_param_errors():
    ctx = lorenz_ctx([1000])
    g = ctx.init_group(LZ_LO, LZ_HI, 1000, 1, 0, seed=5)
    with pytest.raises(FFError) as e:
        ctx.set_param("r", 1000.0)
    assert e.value.status == FF_ERR_RANGE
    with pytest.raises(FFError) as e:
        ctx.set_param("bogus", 1.0)
    assert e.value.status == FF_ERR_UNKNOWN_SYMBOL
    ctx.sweep_param(g, "r", 0.0, 10.0)
    with pytest.raises(FFError) as e:
        ctx.sweep_param(g, "sigma", 0.0, 10.0)
    assert e.value.status == FF_ERR_STATE


# ----------------------------------------------------------------------------- histogram
def special_state(n, rng):
    x = np.vstack([rng.uniform(-12, 12, n), rng.uniform(-35, 35, n), rng.uniform(-5, 55, n)]).astype(np.float32)
    k = n // 20
    x[0, :k] = np.nan
    x[1, k:2 * k] = np.inf
    x[2, 2 * k:3 * k] = -np.inf
    x[0, 3 * k:4 * k] = np.float32(1e-40)     # denormals (FTZ would change these)
    x[1, 3 * k:4 * k] = np.float32(-1e-41)
    x[0, 4 * k:5 * k] = -10.0                 # window edges
    x[0, 5 * k:6 * k] = np.nextafter(np.float32(10.0), np.float32(0))
    x[0, 6 * k:7 * k] = 10.0
    return x


@pytest.mark.parametrize("ppt,tpb", LAUNCHES)
def test_histogram_2d_bit_exact_identical_state(ppt, tpb):
    rng = np.random.default_rng(50)
    n = 40000 + 13
    ctx = lorenz_ctx([n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    x = special_state(n, rng)
    ctx.write_state(g, x)
    view = [-10.0, 10.0, -30.0, 30.0]
    ctx.project([0, 1], view, 333, 211, 2)   # odd sizes, colour 0 of 2 channels
    want = O.histogram(x, [0, 1], view, 333, 211, 2, 0)
    assert np.array_equal(ctx.read_image(), want)


def test_histogram_3d_bit_exact_identical_state():
    rng = np.random.default_rng(51)
    n = 40000 + 13
    ctx = lorenz_ctx([n, n])
    g0 = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    g1 = ctx.init_group(LZ_LO, LZ_HI, n, -1, 1, seed=2)
    x0, x1 = special_state(n, rng), special_state(n, rng)
    x1[1] = rng.uniform(-200, 50, n).astype(np.float32)   # some behind the camera
    ctx.write_state(g0, x0)
    ctx.write_state(g1, x1)
    M = views.lorenz_camera()
    ctx.project([0, 1, 2], M, 1024, 1024, 2)
    want = O.histogram(x0, [0, 1, 2], M, 1024, 1024, 2, 0)
    want = O.histogram(x1, [0, 1, 2], M, 1024, 1024, 2, 1, image=want)
    assert np.array_equal(ctx.read_image(), want)


def test_histogram_collapsed_regime_counts():
    # All particles in one bin (Lorenz r < 1 attractor): counts must still be exact.
    n = 100000
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    ctx.write_state(g, np.zeros((3, n), np.float32))
    img = ctx.project([0, 1], [-1.0, 1.0, -1.0, 1.0], 64, 64, 1)
    im = ctx.read_image()
    assert im.sum() == n and im[0, 32, 32] == n


@pytest.mark.parametrize("ppt,tpb", [(1, 256), (2, 256), (2, 128)])
def test_histogram_aggregation_regimes_exact(ppt, tpb):
    # Runs of 8 equal bins (warp aggregation + block hash table) over ~6k distinct bins (more than
    # the 1024-entry table holds: overflow path), two hot pixels holding half the particles, and
    # scattered particles (direct path) -- all in one image, checked bit-exactly.
    n = 50000 + 3
    rng = np.random.default_rng(52)
    ctx = lorenz_ctx([n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    W, H = 300, 200
    ix = np.repeat(rng.integers(0, W, n // 8 + 1), 8)[:n]
    iy = np.repeat(rng.integers(0, H, n // 8 + 1), 8)[:n]
    hot = rng.random(n) < 0.5
    ix[hot], iy[hot] = np.where(rng.random(hot.sum()) < 0.5, 7, 250), 100
    scat = rng.random(n) < 0.1
    ix[scat], iy[scat] = rng.integers(0, W, scat.sum()), rng.integers(0, H, scat.sum())
    x = np.zeros((3, n), np.float32)
    x[0] = (-10.0 + (ix + 0.5) * (20.0 / W)).astype(np.float32)
    x[1] = (-30.0 + (iy + 0.5) * (60.0 / H)).astype(np.float32)
    ctx.write_state(g, x)
    view = [-10.0, 10.0, -30.0, 30.0]
    ctx.project([0, 1], view, W, H, 1)
    want = O.histogram(x, [0, 1], view, W, H, 1, 0)
    assert np.array_equal(ctx.read_image(), want)
    assert want[0, 100, 7] > n // 5


@pytest.mark.parametrize("ppt,tpb", [(1, 128), (2, 128), (4, 128), (2, 256)])
def test_histogram_warp_regime_with_dropped_leading_lanes(ppt, tpb):
    """Warps whose first lanes hold dropped particles (outside the window) while the others share one
    pixel (the regime is judged on the first lane holding a particle), warps with no particle in view
    at all, and warps in one pixel but for one stray -- bit-exact."""
    n = 4096 * 8 + 5
    ctx = lorenz_ctx([n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    W, H = 64, 48
    idx = np.arange(n)
    x = np.zeros((3, n), np.float32)
    x[0] = -10.0 + 20.0 * (idx % 977 % W + 0.5) / W        # default: scattered
    x[1] = -30.0 + 60.0 * (idx % 331 % H + 0.5) / H
    blk = (idx // 256) % 4
    run = idx % 256
    hot = blk == 0                                           # one pixel, the first 1..31 particles dropped
    x[0, hot], x[1, hot] = -10.0 + 20.0 * 5.5 / W, -30.0 + 60.0 * 7.5 / H
    x[0, hot & (run % 64 < 1 + (idx // 1024) % 31)] = 50.0
    x[0, blk == 1] = 99.0                                    # nothing in view
    stray = blk == 2                                         # one pixel but for one particle
    x[0, stray], x[1, stray] = -10.0 + 20.0 * 40.5 / W, -30.0 + 60.0 * 3.5 / H
    x[1, stray & (run % 64 == 63)] = 20.0
    ctx.write_state(g, x)
    view = [-10.0, 10.0, -30.0, 30.0]
    ctx.project([0, 1], view, W, H, 1)
    want = O.histogram(x, [0, 1], view, W, H, 1, 0)
    assert np.array_equal(ctx.read_image(), want)
    assert want[0, 7, 5] > n // 8


@pytest.mark.parametrize("ppt,tpb", [(0, 0), (4, 128), (2, 256), (2, 128), (1, 128)])
def test_fused_pipeline_matches_oracle_up_to_edge_particles(ppt, tpb):
    """Integrate + bin in one launch vs the oracle's integration and binning, in every launch
    variant: the library default for 30 k particles (one particle per thread), the bench's 4-per-
    thread kernel, and packed pairs in both block sizes."""
    n = 30000
    ctx = lorenz_ctx([n])
    if ppt:
        ctx.set_launch(ppt, tpb)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=2)
    M = views.lorenz_camera()
    img = ctx.project([0, 1, 2], M, 512, 512, 1)
    img.zero_()
    ctx.step(30, 0.01)   # fused: integrate then bin once
    xo = oracle_group(O.LORENZ, LZ_LO, LZ_HI, 2, 0, n, LZ_P, 0.01, 30)
    want = O.histogram(xo, [0, 1, 2], M, 512, 512, 1, 0)
    got = ctx.read_image()
    # particles whose oracle pixel coordinate is within 1e-3 px of a bin edge may land differently
    X = xo.astype(np.float64)
    Md = M.astype(np.float64)
    c = Md @ np.vstack([X, np.ones((1, n))])
    px, py = (c[0] / c[3] + 1) * 256, (c[1] / c[3] + 1) * 256
    near = (np.abs(px - np.round(px)) < 1e-3) | (np.abs(py - np.round(py)) < 1e-3)
    assert np.abs(got.astype(np.int64) - want.astype(np.int64)).sum() <= 2 * near.sum()
    assert got.sum() == want.sum() or abs(int(got.sum()) - int(want.sum())) <= near.sum()


# ----------------------------------------------------------------------------- sharding
def test_shards_sum_to_whole():
    # the image summed over shards equals the unsharded image bit-for-bit.
    n = 25000 + 3
    M = views.lorenz_camera()

    def run(rank, world):
        ctx = FF.Context(systems.lorenz(), [n, n], rank=rank, world=world)
        ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=2)
        ctx.init_group(LZ_LO, LZ_HI, n, -1, 1, seed=3)
        img = ctx.project([0, 1, 2], M, 256, 256, 2)
        img.zero_()
        ctx.step(20, 0.01)
        return ctx.read_image(), [ctx.read_state(k) for k in (0, 1)]

    whole, sw = run(0, 1)
    parts = [run(r, 3) for r in range(3)]
    assert np.array_equal(sum(p[0].astype(np.uint64) for p in parts), whole.astype(np.uint64))
    for k in (0, 1):
        assert np.array_equal(np.hstack([p[1][k] for p in parts]), sw[k])


def test_high_dim_system_compiles_and_matches():
    # 20-D cyclic linear system x_i' = -a x_i + b x_{i+1} exercises the dim > 16 register tiers;
    # checked against the oracle's linear model with the same matrix.
    n_d, a, b = 20, 0.7, 0.3
    s = systems.SystemDef("cyc20", [f"x{i}" for i in range(n_d)],
                          [f"-a*x{i} + b*x{(i + 1) % n_d}" for i in range(n_d)],
                          [("a", a, None, None), ("b", b, None, None)])
    A = np.zeros((n_d, n_d), np.float32)
    for i in range(n_d):
        A[i, i], A[i, (i + 1) % n_d] = -a, b
    ctx = FF.Context(s, [1000])
    g = ctx.init_group([-1.0] * n_d, [1.0] * n_d, 1000, 1, 0, seed=7)
    ctx.step(50, 0.01)
    want = oracle_group(O.LINEAR, [-1.0] * n_d, [1.0] * n_d, 7, 0, 1000, A.ravel(), 0.01, 50)
    assert tier_a(ctx.read_state(g), want, np.ones(n_d)) <= 1e-5


def test_degenerate_inputs():
    """Edge cases of the method: dt = 0 leaves the state bit-identical; a shard that holds no particle
    of a group (world > n) launches, bins nothing and the shards still sum to the whole; a swept group
    next to an unswept one (the latter uses the parameter's value) both match the oracle."""
    n = 4096 + 1
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=21)
    x0 = ctx.read_state(g)
    ctx.step(7, 0.0)
    assert np.array_equal(ctx.read_state(g).view(np.uint32), x0.view(np.uint32))

    # world 3, groups of 2 and 1 particles: some shards hold none of a group
    imgs = []
    for rank in range(3):
        c = FF.Context(systems.lorenz(), [2, 1], rank=rank, world=3)
        c.init_group(LZ_LO, LZ_HI, 2, 1, 0, seed=22)
        c.init_group(LZ_LO, LZ_HI, 1, -1, 1, seed=23)
        img = c.project([0, 2], [-20.0, 20.0, 0.0, 50.0], 64, 64, 2)
        img.zero_()
        c.step(3, 0.01)
        imgs.append(c.read_image().astype(np.uint64))
    whole = np.zeros((2, 64, 64), np.uint64)
    for seed, n_, h, colour in ((22, 2, 0.01, 0), (23, 1, -0.01, 1)):
        x = O.rk4(O.LORENZ, O.ic_uniform(LZ_LO, LZ_HI, seed, 0, n_), LZ_P, np.float32(h), 3)
        whole += O.histogram(x, [0, 2], [-20.0, 20.0, 0.0, 50.0], 64, 64, 2, colour).astype(np.uint64)
    assert np.array_equal(sum(imgs), whole)

    # swept group + unswept group in one context
    m = 6000 + 7
    ctx = lorenz_ctx([m, m], r=20.0)
    gs = ctx.init_group(LZ_LO, LZ_HI, m, 1, 0, seed=24)
    gu = ctx.init_group(LZ_LO, LZ_HI, m, 1, 0, seed=25)
    ctx.sweep_param(gs, "r", 0.0, 40.0, 1)
    sv = O.sweep_values(0.0, 40.0, 1, 0, 0, m, m)
    ctx.step(10, 0.01)
    p = np.array([10.0, 20.0, 8.0 / 3.0], np.float32)
    want_s = O.rk4(O.LORENZ, O.ic_uniform(LZ_LO, LZ_HI, 24, 0, m), p, np.float32(0.01), 10, 1, sv)
    want_u = O.rk4(O.LORENZ, O.ic_uniform(LZ_LO, LZ_HI, 25, 0, m), p, np.float32(0.01), 10)
    assert tier_a(ctx.read_state(gs), want_s, dim_scales(LZ_LO, LZ_HI)) <= 1e-5
    assert tier_a(ctx.read_state(gu), want_u, dim_scales(LZ_LO, LZ_HI)) <= 1e-5


def test_async_state_and_image_copies():
    """ff_write_state_async / ff_read_image_async: stream-ordered copies equal to the synchronous
    ones once the stream is synchronised."""
    from paper_1505_00344_b200 import fireflies as F
    n = 5000 + 3
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=31)
    img = ctx.project([0, 2], [-20.0, 20.0, 0.0, 50.0], 64, 48, 1)
    rng = np.random.default_rng(3)
    src = torch.from_numpy(rng.uniform(-5, 5, (3, n)).astype(np.float32)).pin_memory()
    F.ff_write_state_async(ctx.ctx, g, 0, n, src.data_ptr())
    img.zero_()
    ctx.step(0, 0.01)                              # bins the state just written (stream order)
    out = torch.empty((1, 48, 64), dtype=torch.int32).pin_memory()
    F.ff_read_image_async(ctx.ctx, out.data_ptr())
    ctx.sync()
    assert np.array_equal(ctx.read_state(g), src.numpy())
    assert np.array_equal(out.numpy().view(np.uint32), ctx.read_image())
    assert np.array_equal(ctx.read_image(), O.histogram(src.numpy(), [0, 2], [-20.0, 20.0, 0.0, 50.0], 64, 48, 1, 0))


@pytest.mark.parametrize("W,H,fov,eye,axes", [
    (1280, 720, 60.0, (80.0, -90.0, 60.0), [0, 1, 2]),      # wide image, oblique camera
    (333, 517, 30.0, (0.0, 10.0, 140.0), [2, 0, 1]),        # odd sizes, permuted axes, looking down
])
def test_histogram_3d_other_cameras_bit_exact(W, H, fov, eye, axes):
    """3-D binning with non-square / odd images, other view-projection matrices and permuted axes
    (reading R17-R18), bit-exact vs the oracle on identical coordinates."""
    rng = np.random.default_rng(53)
    n = 30000 + 7
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    x = np.stack([rng.uniform(-40, 40, n), rng.uniform(-60, 60, n), rng.uniform(-10, 80, n)]).astype(np.float32)
    ctx.write_state(g, x)
    Mv = views.look_at(eye, (0.0, 0.0, 25.0), (0.0, 0.0, 1.0) if eye[2] < 100 else (0.0, 1.0, 0.0))
    M = (views.perspective(fov, W / H, 1.0, 1000.0) @ Mv).astype(np.float32)
    ctx.project(axes, M, W, H, 1)
    want = O.histogram(x, axes, M, W, H, 1, 0)
    assert want.sum() > n // 4
    assert np.array_equal(ctx.read_image(), want)


@pytest.mark.parametrize("mode", [0, 1])
def test_swept_shards_sum_to_whole(mode):
    """A swept parameter under sharding: every particle keeps its group-global index,
    so its swept value -- Philox (mode 0) or linspace over the whole group (mode 1) -- and therefore
    its trajectory are the same on any number of shards; the (r, y) images of 3 shards sum to the
    unsharded image bit-for-bit."""
    n = 30000 + 11
    view = [0.0, 200.0, -160.0, 160.0]

    def run(rank, world):
        ctx = FF.Context(systems.lorenz(), [n], rank=rank, world=world)
        g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=5)
        ctx.sweep_param(g, "r", 0.0, 200.0, mode, seed=5)
        img = ctx.project([3, 1], view, 512, 256, 1)
        img.zero_()
        ctx.step(25, 0.01)
        return ctx.read_image().astype(np.uint64), ctx.read_state(g)

    whole, sw = run(0, 1)
    parts = [run(r, 3) for r in range(3)]
    assert np.array_equal(sum(p[0] for p in parts), whole) and whole.sum() > 0
    assert np.array_equal(np.hstack([p[1] for p in parts]).view(np.uint32), sw.view(np.uint32))


@pytest.mark.parametrize("rcpp_stages", [None, "4"])
def test_stn_bifurcation_throughput_variant_sampled(monkeypatch, rcpp_stages):
    """STN-GPe with w_ss swept over [0, 12) (NEXT 4) at a size that selects the
    pipe-balanced throughput kernel (both sigmoids of an evaluation share one reciprocal, on the FMA
    pipe in one of the four stages): sampled slices of both groups, including the ragged tail,
    against the oracle at Tier A after 100 steps; also with the shared reciprocal on the FMA pipe
    (ff_rcpp) in all four stages."""
    if rcpp_stages:
        monkeypatch.setenv("FF_TUNE_RCPP_STAGES", rcpp_stages)
    p, s = stn_params()
    n = 50000 + 19
    ctx = FF.Context(s, [n, n])
    gs = [ctx.init_group([0, 0], [1, 1], n, d, 0, seed=31 + k) for k, d in enumerate((1, -1))]
    for g in gs:
        ctx.sweep_param(g, "w_ss", 0.0, 12.0, 0, 23)
    ctx.step(100, 0.01)
    for k, (g, h) in enumerate(zip(gs, (0.01, -0.01))):
        got = ctx.read_state(g)
        for first, count in ((0, 1500), (24000, 1500), (n - 1501, 1501)):
            sv = O.sweep_values(0.0, 12.0, 0, 23, first, count, n)
            want = oracle_group(O.STN, [0, 0], [1, 1], 31 + k, first, count, p, h, 100, 0, sv)
            assert tier_a(got[:, first:first + count], want, [1.0, 1.0]) <= 1e-5


POISON_CASES = [
    ("stn_bif3d", lambda: systems.stn_gpe(), [0.0, 0.0], [1.0, 1.0], ("w_ss", 0.0, 12.0), [0, 1]),
    ("lorenz_r_swept", lambda: systems.lorenz(), LZ_LO, LZ_HI, ("r", 0.0, 200.0), [0, 2]),
    ("hh_ring3", lambda: systems.hh_ring(3), HH_LO, HH_HI, None, [0, 5]),
]


@pytest.mark.parametrize("name,make,lo,hi,sweep,axes", POISON_CASES, ids=[c[0] for c in POISON_CASES])
def test_poisoned_neighbours_do_not_leak(name, make, lo, hi, sweep, axes):
    """Particles stay independent in the throughput kernel (two particles per thread in packed
    FFMA2 pairs; STN-GPe: clamped sigmoid-pair denominators): with a third of the states replaced by
    NaN, +-inf or +-1e30, every other particle ends bit-identical to the unpoisoned run -- no value,
    and no rounding, crosses between the lanes of a pair (the rejected lane-shared
    reciprocal) -- and the fused binning counts exactly the finite in-window particles."""
    s = make()
    n = 100000 + 3
    rng = np.random.default_rng(60)
    view = [float(lo[axes[0]]), float(hi[axes[0]]), float(lo[axes[1]]), float(hi[axes[1]])]

    def run(x):
        ctx = FF.Context(s, [n])
        g = ctx.init_group(lo, hi, n, 1, 0, seed=41)
        if sweep:
            ctx.sweep_param(g, sweep[0], sweep[1], sweep[2], 0, 23)
        if x is not None:
            ctx.write_state(g, x)
        x0 = ctx.read_state(g)
        ctx.project(axes, view, 256, 256, 1).zero_()
        ctx.step(20, 0.01)
        return x0, ctx.read_state(g), ctx.read_image()

    x0, clean, _ = run(None)
    bad = rng.random(n) < 1 / 3
    poison = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30], np.float32)
    xp = x0.copy()
    xp[:, bad] = poison[rng.integers(0, len(poison), (xp.shape[0], int(bad.sum())))]
    _, dirty, img = run(xp)
    assert np.isfinite(clean).all()
    assert np.array_equal(dirty[:, ~bad].view(np.uint32), clean[:, ~bad].view(np.uint32))
    want = O.histogram(dirty, axes, view, 256, 256, 1, 0)
    assert np.array_equal(img, want)


@pytest.mark.parametrize("seed", list(range(12)))
@pytest.mark.parametrize("ppt,tpb", [(2, 128), (4, 128), (1, 128)])
def test_histogram_3d_random_cameras_and_magnitudes_bit_exact(seed, ppt, tpb):
    """Fuzz of the 3-D binning (reading R18) through the packed pair path (2 and 4 particles per thread:
    FMUL2 / FFMA2 sums, shared reciprocal, ff_div2_pair) and the scalar one: random view-projection
    matrices -- perspective, orthographic-like, and dense random ones with entries over 12 orders of
    magnitude -- and coordinates mixing ordinary values, huge and tiny magnitudes, exact zeros,
    values on pixel edges, infinities and NaN, so both the fast division box and its div.rn fallback
    are hit; the image must equal the oracle's histogram of the same coordinates bit for bit."""
    rng = np.random.default_rng(1000 + seed)
    n = 24000 + seed
    ctx = lorenz_ctx([n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=1)
    W, H = int(rng.integers(17, 700)), int(rng.integers(13, 500))
    kind = seed % 3
    if kind == 0:
        eye = rng.uniform(-150, 150, 3)
        Mv = views.look_at(tuple(eye), tuple(rng.uniform(-10, 10, 3)), (0.0, 0.0, 1.0))
        M = (views.perspective(float(rng.uniform(10, 120)), W / H, 0.1, 5000.0) @ Mv).astype(np.float32)
    elif kind == 1:
        M = np.diag(rng.uniform(0.01, 0.2, 4)).astype(np.float32)
        M[3] = [0.0, 0.0, 0.0, 1.0]
        M[:3, 3] = rng.uniform(-1, 1, 3)
    else:
        M = (rng.standard_normal((4, 4)) * 10.0 ** rng.uniform(-6, 6, (4, 4))).astype(np.float32)
    x = np.stack([rng.uniform(-40, 40, n), rng.uniform(-60, 60, n), rng.uniform(-10, 80, n)]).astype(np.float32)
    pick = rng.random((3, n))
    x[pick < 0.05] *= np.float32(1e25)
    x[(pick >= 0.05) & (pick < 0.10)] *= np.float32(1e-25)
    x[(pick >= 0.10) & (pick < 0.12)] = 0.0
    x[(pick >= 0.12) & (pick < 0.13)] = np.inf
    x[(pick >= 0.13) & (pick < 0.14)] = -np.inf
    x[(pick >= 0.14) & (pick < 0.15)] = np.nan
    ctx.write_state(g, x)
    ctx.project([0, 1, 2], M, W, H, 1)
    want = O.histogram(x, [0, 1, 2], M, W, H, 1, 0)
    got = ctx.read_image()
    assert np.array_equal(got, want), f"{np.count_nonzero(got != want)} pixels differ (kind {kind})"


def test_swept_lorenz_lands_on_the_pitchfork_branches():
    """Closed-form pin of the whole swept path (no oracle in the loop): configs[3]'s shape with r
    Philox-swept over [0, 13) (2^20 particles, the bench's 4-per-thread kernel, 1000-step launches).
    PAPER.md:89, :95: below r = 1 every particle goes to the origin (checked for r < 0.5); between the pitchfork and the
    homoclinic r = 13.926 at C+- = (+-sqrt(8(r-1)/3), +-sqrt(8(r-1)/3), r - 1) -- each particle at the
    fixed points of its OWN r (read back with ff_read_lifted), after 5000 RK4 steps."""
    n = 1 << 20
    ctx = lorenz_ctx([n])
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=31)
    ctx.sweep_param(g, "r", 0.0, 13.0, 0, seed=32)
    for _ in range(5):
        ctx.step(1000, 0.01)
    x = ctx.read_state(g).astype(np.float64)
    r = ctx.read_lifted(g).astype(np.float64)
    assert np.array_equal(r.astype(np.float32), O.sweep_values(0.0, 13.0, 0, 32, 0, n, n))
    low = r < 0.5          # (the origin's slowest rate, (sqrt(81 + 40 r) - 11) / 2, is -0.48 at r = 0.5)
    assert low.sum() > 30000 and np.abs(x[:, low]).max() < 1e-3
    mid = (r > 1.5) & (r < 12.5)
    c = np.sqrt(8.0 / 3.0 * (r[mid] - 1.0))
    assert mid.sum() > 700000
    # (a particle starting next to the z axis -- the saddle's stable manifold -- lingers there for
    # ln(1/distance) / 0.44 time units, so a handful of the 2^20 may still be on their way at t = 50)
    dev = np.maximum(np.abs(np.abs(x[0, mid]) - c), np.abs(np.abs(x[1, mid]) - c)) / c
    dev = np.maximum(dev, np.abs(x[2, mid] - (r[mid] - 1.0)) / (r[mid] - 1.0))
    assert np.mean(dev < 1e-4) > 0.9999, np.sort(dev)[-10:]
    assert np.all(np.sign(x[0, mid]) == np.sign(x[1, mid]))          # C+ or C-, never mixed
    assert np.isfinite(x).all() and np.abs(x).max() < 60.0
    both = np.mean(x[0, mid] > 0)
    assert 0.3 < both < 0.7                                            # both branches populated
