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
