"""Pins of the oracle's reset rule (reading R16) -- no GPU."""
import numpy as np

import oracle as O


def fresh(n, seed=3):
    return O.ic_uniform([0.0, 0.0], [1.0, 1.0], seed, 0, n), np.zeros(n, np.float32), np.zeros(n, np.uint32)


def test_in_bounds_untouched_bit_exact():
    x, b, e = fresh(1000)
    x0 = x.copy()
    O.reset(x, [0, 0], [1, 1], 0.0, 5.0, b, e, [0, 0], [1, 1], 3)
    assert np.array_equal(x, x0) and not e.any() and not b.any()


def test_escaped_particles_get_new_box_draws():
    # "Any trajectories that leave this square region ... are reset to a new random set of initial
    # conditions": every escaped particle lands back in the IC box, others unchanged.
    x, b, e = fresh(5000)
    rng = np.random.default_rng(0)
    out = rng.random(5000) < 0.3
    x[0, out] += 1.5
    x[1, rng.random(5000) < 0.01] = np.nan
    bad = out | np.isnan(x[1])
    x0 = x.copy()
    O.reset(x, [0, 0], [1, 1], 0.0, 2.5, b, e, [0, 0], [1, 1], 3)
    assert np.array_equal(e.astype(bool), bad)
    assert np.all(b[bad] == 2.5) and np.all(b[~bad] == 0)
    assert np.all((x[:, bad] >= 0) & (x[:, bad] < 1))
    assert np.array_equal(x[:, ~bad], x0[:, ~bad])
    # the redraw is not the particle's original initial condition (stream 2 + epoch != stream 0)
    orig = O.ic_uniform([0.0, 0.0], [1.0, 1.0], 3, 0, 5000)
    assert not np.any(np.all(x[:, bad] == orig[:, bad], axis=0))


def test_bounds_edges_inclusive_and_nonfinite_only_mode():
    x = np.array([[0.0, 1.0, np.nextafter(np.float32(1), np.float32(2)), -0.0, np.inf]], np.float32)
    b, e = np.zeros(5, np.float32), np.zeros(5, np.uint32)
    O.reset(x, [0.0], [1.0], 0.0, 1.0, b, e, [0.0], [1.0], 1)
    assert list(e) == [0, 0, 1, 0, 1]
    x = np.array([[5.0, -1e30, np.nan, np.inf, -np.inf]], np.float32)
    b, e = np.zeros(5, np.float32), np.zeros(5, np.uint32)
    O.reset(x, None, None, 0.0, 1.0, b, e, [0.0], [1.0], 1)
    assert list(e) == [0, 0, 1, 1, 1]


def test_age_rule_and_epochs_advance():
    # "... or which have not been reset for more than time T_max"
    x, b, e = fresh(100)
    b[:50] = 0.0
    b[50:] = 4.0
    O.reset(x, [0, 0], [1, 1], 5.0, 6.0, b, e, [0, 0], [1, 1], 3)   # ages 6 (> 5) and 2
    assert e[:50].all() and not e[50:].any()
    first = x[:, :50].copy()
    x[0, :50] = 7.0   # leave again: second reset uses stream 2 + 1, a different draw
    O.reset(x, [0, 0], [1, 1], 5.0, 6.5, b, e, [0, 0], [1, 1], 3)
    assert np.all(e[:50] == 2) and not np.any(np.all(x[:, :50] == first, axis=0))


def test_reset_draws_uniform_in_box():
    n = 100000
    x = np.full((2, n), np.nan, np.float32)
    b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
    O.reset(x, None, None, 0.0, 1.0, b, e, [-2.0, 10.0], [2.0, 20.0], 9)
    for d, (lo, hi) in enumerate(((-2.0, 2.0), (10.0, 20.0))):
        u = np.sort((x[d].astype(np.float64) - lo) / (hi - lo))
        assert np.max(np.abs(np.arange(1, n + 1) / n - u)) < 0.01


# ---- the lifted (swept) parameter is redrawn with the state (reading R16)

import json
import os

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_independent_philox_reproduces_known_answers():
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen_reset_golden", os.path.join(GOLD, "gen_reset_golden.py"))
    g = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(g)
    g.check_kat()   # the golden file's generator is a correct Philox4x32-10


def test_reset_redraw_bits_match_independent_golden():
    """Every reset redraw word / value (state and lifted component) equals the golden file written by
    an independent pure-Python Philox (tests/golden/gen_reset_golden.py)."""
    doc = json.load(open(os.path.join(GOLD, "reset_golden.json")))
    for c in doc["cases"]:
        dim = len(c["lo"])
        x = np.full((dim, 1), np.nan, np.float32)
        b, e = np.zeros(1, np.float32), np.array([c["reset"]], np.uint32)
        sweep = None
        if "sweep" in c:
            sv = np.array([-123.0], np.float32)
            sweep = dict(vals=sv, lo=c["sweep"][0], hi=c["sweep"][1], mode=0, seed=999, n_group=c["index"] + 1)
        O.reset(x, None, None, 0.0, 1.0, b, e, c["lo"], c["hi"], c["seed"], first_global=c["index"], sweep=sweep)
        assert e[0] == c["reset"] + 1
        got = ["%08x" % int(v) for v in x[:, 0].view(np.uint32)]
        assert got == c["bits"], c
        for d in range(dim):   # the oracle's own Philox gives the golden words for every component
            w = O.philox4x32_10([c["index"] & 0xffffffff, c["index"] >> 32, d // 4, 2 + c["reset"]],
                                [c["seed"] & 0xffffffff, c["seed"] >> 32])
            assert "%08x" % int(w[d % 4]) == c["words"][d]
        if sweep is not None:
            assert "%08x" % int(sv.view(np.uint32)[0]) == c["lifted_bits"], c
            lv = O.lifted_values(c["sweep"][0], c["sweep"][1], 0, 999, c["seed"], dim, c["index"], 1,
                                 c["index"] + 1, [c["reset"] + 1])
            assert lv.view(np.uint32)[0] == sv.view(np.uint32)[0]


def test_lifted_value_epoch0_is_the_sweep_draw_and_linspace_stays_fixed():
    n = 4000
    for mode in (0, 1):
        base = O.sweep_values(0.0, 12.0, mode, 23, 100, n, 10 * n)
        assert np.array_equal(O.lifted_values(0.0, 12.0, mode, 23, 22, 2, 100, n, 10 * n), base)
        x, b, e = fresh(n, seed=22)
        x[0, ::3] = 5.0   # a third leave the unit square
        sv = base.copy()
        O.reset(x, [0, 0], [1, 1], 0.0, 1.0, b, e, [0, 0], [1, 1], 22, first_global=100,
                sweep=dict(vals=sv, lo=0.0, hi=12.0, mode=mode, seed=23, n_group=10 * n))
        moved = e.astype(bool)
        assert moved.sum() == len(range(0, n, 3))
        assert np.array_equal(sv[~moved], base[~moved])
        if mode == 1:   # linspace: a grid, not a random initial condition -- fixed through resets
            assert np.array_equal(sv, base)
        else:
            assert not np.any(sv[moved] == base[moved])
            assert np.all((sv >= 0) & (sv < 12))
        assert np.array_equal(O.lifted_values(0.0, 12.0, mode, 23, 22, 2, 100, n, 10 * n, e), sv)


def test_reset_lifted_draws_uniform_and_weight_long_lived_values():
    """The redraw is uniform over the swept range (the IC range of the lifted variable);
    so particles whose parameter value makes them escape often spend less time at that value: after
    repeated resets of only the particles with w > 6, the time-averaged share of w < 6 grows."""
    n = 200000
    x = np.full((2, n), np.nan, np.float32)
    b, e = np.zeros(n, np.float32), np.zeros(n, np.uint32)
    sv = O.sweep_values(0.0, 12.0, 0, 7, 0, n, n)
    O.reset(x, None, None, 0.0, 1.0, b, e, [0, 0], [1, 1], 8, sweep=dict(vals=sv, lo=0.0, hi=12.0, mode=0, seed=7))
    u = np.sort(sv.astype(np.float64) / 12.0)
    assert np.max(np.abs(np.arange(1, n + 1) / n - u)) < 0.006
    shares = []
    for k in range(4):
        x[:, sv > 6.0] = np.nan   # only large-w particles escape
        O.reset(x, None, None, 0.0, 2.0 + k, b, e, [0, 0], [1, 1], 8,
                sweep=dict(vals=sv, lo=0.0, hi=12.0, mode=0, seed=7))
        shares.append(np.mean(sv < 6.0))
    assert shares[0] > 0.7 and all(b > a for a, b in zip(shares, shares[1:]))   # 3/4, 7/8, ...
