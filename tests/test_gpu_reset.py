"""GPU parity of the device-side reset (NEXT row 1) against the oracle's
reset rule, through the C ABI."""
import numpy as np
import pytest

import oracle as O
from parity import dim_scales, scaled_error

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402


def stn_params():
    s = systems.stn_gpe()
    return s, np.array([p[1] for p in s.params], np.float32)


@pytest.mark.parametrize("ppt,tpb", [(1, 256), (2, 256)])
def test_stn_backward_reset_to_unit_square(ppt, tpb):
    # backward STN particles leave (0,1)^2 and are reset to new random ICs.
    s, p = stn_params()
    n, S, seed = 8000 + 11, 40, 11
    ctx = FF.Context(s, [n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group([0, 0], [1, 1], n, -1, 0, seed=seed)
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)
    x = O.ic_uniform([0, 0], [1, 1], seed, 0, n)
    b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
    t = 0.0
    mismatched = 0
    for launch in range(4):
        ctx.step(S, 0.01)
        t += abs(float(np.float32(0.01))) * S
        x = O.rk4(O.STN, x, p, np.float32(-0.01), S)
        e_before = e.copy()
        O.reset(x, [0, 0], [1, 1], 0.0, np.float32(t), b, e, [0, 0], [1, 1], seed)
        got, ge = ctx.read_state(g), ctx.read_epochs(g)
        same = ge == e
        # decision mismatches only where the oracle state sat within 1e-4 of the square's edge
        mismatched += int((~same).sum())
        assert (~same).sum() <= max(2, n // 1000)
        fresh = same & (e != e_before)
        assert np.array_equal(got[:, fresh].view(np.uint32), x[:, fresh].view(np.uint32))  # bit-exact redraws
        keep = same & (e == e_before) & (e == 0)
        err = scaled_error(got[:, keep], x[:, keep], [1.0, 1.0])
        assert err.size == 0 or err.max() <= 1e-5
        # resync the oracle to the GPU where the decision differed (test logic, not oracle input)
        x[:, ~same], e[~same] = got[:, ~same], ge[~same]
        assert np.all((got >= 0) & (got <= 1)), "after a reset launch every particle is inside the square"
    assert e.sum() > n  # most particles were reset at least once


def test_lorenz_backward_nonfinite_reset():
    # Backward Lorenz particles blow up; non-finite particles are reset (no bounds).
    lo, hi = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]
    p = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
    n, seed = 20000, 3
    ctx = FF.Context(systems.lorenz(), [n])
    g = ctx.init_group(lo, hi, n, -1, 0, seed=seed)
    ctx.set_reset(True)
    ctx.step(200, 0.01)
    x = O.rk4(O.LORENZ, O.ic_uniform(lo, hi, seed, 0, n), p, np.float32(-0.01), 200)
    b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
    O.reset(x, None, None, 0.0, np.float32(2.0), b, e, lo, hi, seed)
    got, ge = ctx.read_state(g), ctx.read_epochs(g)
    assert np.all(np.isfinite(got))
    assert ge.sum() > n // 2
    same = ge == e
    assert (~same).sum() <= n // 1000
    fresh = same & (e == 1)
    assert np.array_equal(got[:, fresh].view(np.uint32), x[:, fresh].view(np.uint32))


def test_age_reset_all_particles():
    n = 3000
    ctx = FF.Context(systems.lorenz(), [n])
    g = ctx.init_group([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], n, 1, 0, seed=4)
    ctx.set_reset(True, None, None, 0.05)   # T_max = 0.05 time units = 5 steps
    ctx.step(3, 0.01)
    assert not ctx.read_epochs(g).any()
    ctx.step(3, 0.01)                        # age 0.06 > 0.05: everyone resets
    assert np.all(ctx.read_epochs(g) == 1)
    x = O.ic_uniform([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], 4, 0, n)
    b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
    O.reset(x, None, None, 0.05, np.float32(6 * float(np.float32(0.01))), b, e,
            [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0], 4)
    assert np.array_equal(ctx.read_state(g).view(np.uint32), x.view(np.uint32))


def test_stn_bifurcation_3d_pipeline():
    # NEXT row 4: w_ss lifted (swept per particle over [0, 12)), forward and
    # backward groups, reset to the unit square, 3-D projection of (x, y, w_ss). One fused launch of
    # 100 steps + reset + binning, checked against oracle integration + reset + histogram.
    s, p = stn_params()
    n = 6000 + 7
    ctx = FF.Context(s, [n, n])
    gf = ctx.init_group([0, 0], [1, 1], n, 1, 0, seed=21)
    gb = ctx.init_group([0, 0], [1, 1], n, -1, 1, seed=22)
    for g in (gf, gb):
        ctx.sweep_param(g, "w_ss", 0.0, 12.0, 0, 23)
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)
    M = views.box_camera([0.0, 0.0, 0.0], [1.0, 1.0, 12.0])
    img = ctx.project([0, 1, 2], M, 256, 256, 2)
    img.zero_()
    ctx.step(100, 0.01)
    sv = O.sweep_values(0.0, 12.0, 0, 23, 0, n, n)
    want_img = np.zeros((2, 256, 256), np.uint32)
    t = np.float32(abs(float(np.float32(0.01))) * 100)
    for g, seed, h, ch in ((gf, 21, 0.01, 0), (gb, 22, -0.01, 1)):
        x = O.rk4(O.STN, O.ic_uniform([0, 0], [1, 1], seed, 0, n), p, np.float32(h), 100, 0, sv)
        b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
        svg = sv.copy()   # reset particles redraw their w_ss too (reading R16)
        O.reset(x, [0, 0], [1, 1], 0.0, t, b, e, [0, 0], [1, 1], seed,
                sweep=dict(vals=svg, lo=0.0, hi=12.0, mode=0, seed=23, n_group=n))
        got, ge = ctx.read_state(g), ctx.read_epochs(g)
        same = ge == e
        assert (~same).sum() <= 3
        err = scaled_error(got[:, same], x[:, same], [1.0, 1.0])
        assert err.max() <= 1e-5
        lifted = ctx.read_lifted(g)
        assert np.array_equal(lifted[same].view(np.uint32), svg[same].view(np.uint32))
        if ch == 1:
            assert (e > 0).mean() > 0.5 and np.any(svg != sv)   # backward particles escape and redraw
        O.histogram(x, [0, 1, 2], M, 256, 256, 2, ch, image=want_img, sweep_vals=svg)
    got_img = ctx.read_image().astype(np.int64)
    # particles near a pixel edge (or with a different reset decision) may land one bin apart
    assert np.abs(got_img - want_img.astype(np.int64)).sum() <= 2 * 40
    assert got_img.sum() == want_img.sum()


def test_reset_then_binning_sees_new_positions():
    # the fused binning runs after the reset: every particle of a collapsed backward group counts
    s, p = stn_params()
    n = 4096
    ctx = FF.Context(s, [n])
    ctx.init_group([0, 0], [1, 1], n, -1, 0, seed=2)
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)
    img = ctx.project([0, 1], [0.0, 1.0, 0.0, 1.0], 64, 64, 1)
    for _ in range(5):
        img.zero_()
        ctx.step(100, 0.01)
        assert int(ctx.read_image().sum()) == n


@pytest.mark.parametrize("mode", [0, 1])
def test_lifted_values_readback_epoch0(mode):
    # before any reset the lifted value is the sweep draw (reading R13), bit-exact
    s, _ = stn_params()
    n = 5000 + 3
    ctx = FF.Context(s, [n])
    g = ctx.init_group([0, 0], [1, 1], n, 1, 0, seed=9)
    ctx.sweep_param(g, "w_ss", 0.0, 12.0, mode, 31)
    want = O.sweep_values(0.0, 12.0, mode, 31, 0, n, n)
    assert np.array_equal(ctx.read_lifted(g).view(np.uint32), want.view(np.uint32))
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)   # bookkeeping exists, every epoch 0
    assert np.array_equal(ctx.read_lifted(g).view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("ppt,tpb", [(1, 128), (2, 256), (4, 128)])
@pytest.mark.parametrize("mode", [0, 1])
def test_reset_redraws_lifted_parameter(ppt, tpb, mode):
    """PAPER.md:54 / :207: the swept parameter is a state variable whose IC range is the sweep range,
    and a reset draws a new position -- so a reset particle gets a new w_ss (mode 0), bit-exact vs
    the oracle's reset rule; non-reset particles keep theirs; the state keeps Tier A with the new
    values; the fused image bins (x, w_ss) with them. Linspace sweeps (mode 1) keep their grid value."""
    s, p = stn_params()
    n, S, seed, sseed = 8000 + 13, 50, 22, 23
    ctx = FF.Context(s, [n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group([0, 0], [1, 1], n, -1, 0, seed=seed)
    ctx.sweep_param(g, "w_ss", 0.0, 12.0, mode, sseed)
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)
    view = [0.0, 1.0, 0.0, 12.0]
    img = ctx.project([0, 2], view, 128, 96, 1)
    x = O.ic_uniform([0, 0], [1, 1], seed, 0, n)
    sv = O.sweep_values(0.0, 12.0, mode, sseed, 0, n, n)
    sv0 = sv.copy()
    b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
    t = 0.0
    for launch in range(3):
        img.zero_()
        ctx.step(S, 0.01)
        t += abs(float(np.float32(0.01))) * S
        x = O.rk4(O.STN, x, p, np.float32(-0.01), S, 0, sv)
        e_before = e.copy()
        O.reset(x, [0, 0], [1, 1], 0.0, np.float32(t), b, e, [0, 0], [1, 1], seed,
                sweep=dict(vals=sv, lo=0.0, hi=12.0, mode=mode, seed=sseed, n_group=n))
        got, ge, lifted = ctx.read_state(g), ctx.read_epochs(g), ctx.read_lifted(g)
        # the GPU's lifted values are the oracle's function of the GPU's own epochs, for every particle
        want_l = O.lifted_values(0.0, 12.0, mode, sseed, seed, 2, 0, n, n, ge)
        assert np.array_equal(lifted.view(np.uint32), want_l.view(np.uint32))
        same = ge == e
        assert (~same).sum() <= max(2, n // 1000)
        assert np.array_equal(lifted[same].view(np.uint32), sv[same].view(np.uint32))
        fresh = same & (e != e_before)
        assert np.array_equal(got[:, fresh].view(np.uint32), x[:, fresh].view(np.uint32))
        if mode == 1:
            assert np.array_equal(lifted.view(np.uint32), sv0.view(np.uint32))
        elif launch == 0:
            assert np.all(lifted[fresh] != sv0[fresh]) and fresh.sum() > n // 4
        keep = same & (e == e_before)
        err = scaled_error(got[:, keep], x[:, keep], [1.0, 1.0])
        assert err.size == 0 or err.max() <= 1e-5
        # fused image of (x, w_ss) after the reset == the oracle's binning of the GPU's state and lifted
        # values (P3: identical coordinates -> bit-exact)
        want_img = O.histogram(got, [0, 2], view, 128, 96, 1, 0, sweep_vals=lifted)
        assert np.array_equal(ctx.read_image(), want_img)
        x[:, ~same], e[~same], sv[~same] = got[:, ~same], ge[~same], lifted[~same]   # resync (test logic)
    # disabling and re-enabling the reset rule keeps every particle's lifted value
    before = ctx.read_lifted(g)
    ctx.set_reset(False)
    ctx.set_reset(True, [0.0, 0.0], [1.0, 1.0], 0.0)
    assert np.array_equal(ctx.read_lifted(g).view(np.uint32), before.view(np.uint32))


def test_lifted_redraw_uses_a_second_philox_block_at_dim_4():
    # a 4-variable system: the lifted component is word 0 of Philox block 1 (tests/golden reset_golden)
    import json
    import os
    doc = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reset_golden.json")))
    case = [c for c in doc["cases"] if len(c["lo"]) == 4][0]
    from paper_1505_00344_b200.systems import SystemDef
    sysdef = SystemDef("lin4", ["a", "b", "c", "d"], ["k*a", "k*b", "k*c", "k*d"], [("k", 0.0, None, None)])
    n = case["index"] + 1
    ctx = FF.Context(sysdef, [n])
    g = ctx.init_group(case["lo"], case["hi"], n, 1, 0, seed=case["seed"])
    ctx.sweep_param(g, "k", case["sweep"][0], case["sweep"][1], 0, 77)
    ctx.set_reset(True)
    for r in range(case["reset"] + 1):   # poison the particle once per launch: e resets -> epoch e + 1
        st = ctx.read_state(g)
        st[:, case["index"]] = np.nan
        ctx.write_state(g, st)
        ctx.step(1, 0.0)
    assert ctx.read_epochs(g)[case["index"]] == case["reset"] + 1
    got = ctx.read_state(g)[:, case["index"]]
    assert ["%08x" % v for v in got.view(np.uint32)] == case["bits"]
    assert "%08x" % ctx.read_lifted(g)[case["index"]:].view(np.uint32)[0] == case["lifted_bits"]


@pytest.mark.parametrize("dim,ppt,tpb,steps", [(4, 1, 128, 1), (4, 2, 128, 1), (4, 2, 256, 1), (4, 4, 128, 1),
                                               (4, 4, 128, 60), (9, 1, 128, 1), (9, 2, 128, 1), (9, 2, 128, 60)])
@pytest.mark.parametrize("density", [0.01, 0.2, 0.95])
def test_redraws_bit_exact_at_any_reset_density(dim, ppt, tpb, steps, density):
    """The redraw is warp-cooperative when a warp has few resets (jobs spread over the lanes, results
    shuffled back; 4-per-thread launches of >= 50 steps redraw per thread instead): both must give the
    oracle's bits. Particles of a 4- or 9-variable system with a Philox-swept lifted parameter (its
    redraw needs a second / third Philox block; 9 variables shuffle 10 values per job) are poisoned
    with NaN at random at the given density and stepped with dt = 0 (nothing else moves; 60 steps
    select the long-launch build): every poisoned particle is redrawn exactly as the oracle's reset
    rule with its epoch
    (state and lifted value), every other one keeps its bits."""
    from paper_1505_00344_b200.systems import SystemDef
    names = ["v%d" % d for d in range(dim)]
    sysdef = SystemDef("lin%d" % dim, names, ["k*" + v for v in names], [("k", 0.0, None, None)])
    lo = ([-1.0, 0.0, 2.0, -5.0] * 3)[:dim]
    hi = ([1.0, 3.0, 2.5, 5.0] * 3)[:dim]
    seed, sseed = 31, 77
    n = 20000 + 37
    ctx = FF.Context(sysdef, [n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(lo, hi, n, 1, 0, seed=seed)
    ctx.sweep_param(g, "k", 0.5, 1.5, 0, sseed)
    ctx.set_reset(True)
    rng = np.random.default_rng(int(density * 1000) + ppt)
    prev_ep = np.zeros(n, np.uint32)
    for _ in range(3):
        before, lifted0 = ctx.read_state(g), ctx.read_lifted(g)
        sel = rng.random(n) < density
        st = before.copy()
        st[:, sel] = np.nan
        ctx.write_state(g, st)
        ctx.step(steps, 0.0)
        ep, got, lifted = ctx.read_epochs(g), ctx.read_state(g), ctx.read_lifted(g)
        assert np.array_equal(ep, prev_ep + sel.astype(np.uint32))
        keep = ~sel
        assert np.array_equal(got[:, keep].view(np.uint32), before[:, keep].view(np.uint32))
        assert np.array_equal(lifted[keep].view(np.uint32), lifted0[keep].view(np.uint32))
        for i in np.nonzero(sel)[0]:
            col = np.full((dim, 1), np.nan, np.float32)
            sv = np.zeros(1, np.float32)
            O.reset(col, None, None, 0.0, 0.0, np.zeros(1, np.float32), np.array([ep[i] - 1], np.uint32), lo, hi,
                    seed, first_global=int(i), sweep=dict(vals=sv, lo=0.5, hi=1.5, mode=0, seed=sseed, n_group=n))
            assert np.array_equal(got[:, i].view(np.uint32), col[:, 0].view(np.uint32)), i
            assert sv.view(np.uint32)[0] == lifted[i:i + 1].view(np.uint32)[0], i
        prev_ep = ep
