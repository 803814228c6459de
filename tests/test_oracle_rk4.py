"""Pins of the oracle's RK4 integrator against closed forms and properties the mathematics fixes
(no GPU). The oracle's RK4 follows PAPER.md:42 ("4th order Runge-Kutta", constant step) with the
classical tableau (reading R1)."""
import numpy as np
import pytest

import oracle as O


def T4(z):
    """Stability polynomial of classical RK4: exact one-step map of x' = a x is x -> T4(h a) x."""
    return 1 + z + z ** 2 / 2 + z ** 3 / 6 + z ** 4 / 24


def test_linear_one_step_hand_values():
    # SPEC.md:254 (x'=-x, x=1, h=0.1 -> 0.9048375) and :256 (h=-0.1 -> 1.1051708...).
    x = O.rk4(O.LINEAR, np.array([[1.0]]), [-1.0], 0.1, 1)
    assert x[0, 0] == pytest.approx(0.9048375, abs=1e-15)
    x = O.rk4(O.LINEAR, np.array([[1.0]]), [-1.0], -0.1, 1)
    assert x[0, 0] == pytest.approx(1.1051708333333333, abs=1e-15)


@pytest.mark.parametrize("h", [0.1, -0.05, 0.013])
def test_linear_matrix_closed_form(h):
    # For x' = A x the RK4 map is exactly T4(hA); compare n steps against the matrix power.
    rng = np.random.default_rng(1)
    A = rng.normal(size=(4, 4))
    x0 = rng.normal(size=(4, 5))
    n = 17
    M = np.eye(4) + h * A + (h * A) @ (h * A) / 2 + np.linalg.matrix_power(h * A, 3) / 6 + \
        np.linalg.matrix_power(h * A, 4) / 24
    want = np.linalg.matrix_power(M, n) @ x0
    got = O.rk4(O.LINEAR, x0, A.ravel(), h, n)
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


def test_order_four_convergence_linear():
    # global error at t=1 of x'=-x shrinks by 12..20x per halving of h.
    errs = []
    for h in (0.1, 0.05, 0.025):
        n = int(round(1 / h))
        x = O.rk4(O.LINEAR, np.array([[1.0]]), [-1.0], h, n)
        errs.append(abs(x[0, 0] - np.exp(-1.0)))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 12 <= r1 <= 20 and 12 <= r2 <= 20


def test_order_four_self_convergence_lorenz():
    # Nonlinear check of the tableau: successive differences shrink by ~16 per halving.
    x0 = np.array([[1.0], [1.0], [1.0]])
    p = [10.0, 28.0, 8.0 / 3.0]
    sols = []
    for k in range(4):
        h = 0.01 / 2 ** k
        sols.append(O.rk4(O.LORENZ, x0, p, h, 50 * 2 ** k)[:, 0])
    d1 = np.linalg.norm(sols[0] - sols[1])
    d2 = np.linalg.norm(sols[1] - sols[2])
    d3 = np.linalg.norm(sols[2] - sols[3])
    assert 12 <= d1 / d2 <= 20 and 12 <= d2 / d3 <= 20


def test_harmonic_radius_closed_form():
    # For rotation the per-step radius factor is |T4(i h)| = sqrt(1 - h^6/72 + h^8/576);
    # SPEC.md:303 (drift < 1e-6 per period at h = 0.01).
    h = 0.01
    n = int(round(2 * np.pi / h))
    x = O.rk4(O.HARMONIC, np.array([[1.0], [0.0]]), [1.0], h, n)
    r = np.hypot(x[0, 0], x[1, 0])
    want = abs(T4(1j * h)) ** n
    assert r == pytest.approx(want, abs=1e-13)
    assert abs(r - 1) < 1e-6


def test_round_trip_linear():
    # Phi_{-h} o Phi_h = T4(z) T4(-z) on x' = a x.
    a, h = -0.7, 0.2
    x = O.rk4(O.LINEAR, np.array([[1.0]]), [a], h, 1)
    x = O.rk4(O.LINEAR, x, [a], -h, 1)
    z = a * h
    assert x[0, 0] == pytest.approx(T4(z) * T4(-z), abs=1e-15)


def test_round_trip_lorenz_short():
    # Nonlinear: forward then backward 10 steps returns within O(h^5)-sized error.
    rng = np.random.default_rng(2)
    x0 = np.vstack([rng.uniform(-10, 10, 50), rng.uniform(-30, 30, 50), rng.uniform(0, 50, 50)])
    p = [10.0, 28.0, 8.0 / 3.0]
    x = O.rk4(O.LORENZ, O.rk4(O.LORENZ, x0, p, 0.001, 10), p, -0.001, 10)
    np.testing.assert_allclose(x, x0, atol=1e-9)


def test_zero_rhs_is_identity():
    # SPEC.md:255 (x' = 0 -> x unchanged), bit-exactly.
    x0 = np.array([[1.2345], [-7.5]], dtype=np.float32)
    x = O.rk4(O.LINEAR, x0, np.zeros(4, dtype=np.float32), 0.01, 1000)
    assert np.array_equal(x, x0)


def test_fixed_point_origin_bit_exact():
    # the origin is a fixed point of Lorenz for every r; f = 0 exactly there.
    x = O.rk4(O.LORENZ, np.zeros((3, 1), dtype=np.float32), np.array([10, 28, 8 / 3], np.float32), 0.01, 500)
    assert np.all(x == 0)


def test_swept_parameter_per_particle():
    # each particle carries its own fixed value of the lifted parameter.
    # Running a block of particles with per-particle r must equal running each alone.
    rng = np.random.default_rng(3)
    x0 = np.vstack([rng.uniform(-10, 10, 8), rng.uniform(-30, 30, 8), rng.uniform(0, 50, 8)])
    rs = rng.uniform(0, 200, 8)
    got = O.rk4(O.LORENZ, x0, [10.0, 0.0, 8 / 3], 0.01, 30, sweep_idx=1, sweep_vals=rs)
    for i in range(8):
        one = O.rk4(O.LORENZ, x0[:, i:i + 1], [10.0, rs[i], 8 / 3], 0.01, 30)
        assert np.array_equal(got[:, i], one[:, 0])


def test_permutation_invariance_and_independence():
    # permuting particles permutes results (no cross-particle coupling).
    rng = np.random.default_rng(4)
    x0 = np.vstack([rng.uniform(-10, 10, 64), rng.uniform(-30, 30, 64), rng.uniform(0, 50, 64)]).astype(np.float32)
    p = np.array([10, 28, 8 / 3], np.float32)
    perm = rng.permutation(64)
    a = O.rk4(O.LORENZ, x0, p, np.float32(0.01), 20)
    b = O.rk4(O.LORENZ, x0[:, perm], p, np.float32(0.01), 20)
    assert np.array_equal(a[:, perm], b)


def test_f32_tracks_f64_short_horizon():
    rng = np.random.default_rng(5)
    x0 = np.vstack([rng.uniform(-10, 10, 200), rng.uniform(-30, 30, 200), rng.uniform(0, 50, 200)])
    p = [10.0, 28.0, 8 / 3]
    a = O.rk4(O.LORENZ, x0.astype(np.float32), np.array(p, np.float32), 0.01, 20)
    b = O.rk4(O.LORENZ, x0, p, 0.01, 20)
    np.testing.assert_allclose(a, b, atol=1e-4 * 50)


def test_bad_arguments_rejected():
    with pytest.raises(ValueError):
        O.rk4(99, np.zeros((3, 1)), [1.0], 0.1, 1)
    with pytest.raises(ValueError):
        O.rk4(O.LORENZ, np.zeros((4, 1)), [1.0, 1.0, 1.0], 0.1, 1)
