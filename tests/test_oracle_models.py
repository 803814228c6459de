"""Pins of the oracle's hand-coded right-hand sides against what the paper states and what the
mathematics of each model fixes (no GPU)."""
import json
import os

import numpy as np
import pytest
from scipy.special import expit

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
LORENZ_P = [10.0, 28.0, 8.0 / 3.0]


def lorenz_box(n, seed):
    rng = np.random.default_rng(seed)
    # Fig. 3A IC box.
    return np.vstack([rng.uniform(-10, 10, n), rng.uniform(-30, 30, n), rng.uniform(0, 50, n)])


# ----------------------------------------------------------------------------- Lorenz
def test_lorenz_rhs_hand_value():
    # rhs(1,1,1) with sigma=10, r=28, beta=8/3 is (0, 26, -5/3) -- direct
    # substitution into PAPER.md Eqs. 3-5.
    np.testing.assert_allclose(O.rhs(O.LORENZ, [1, 1, 1], LORENZ_P), [0, 26, -5 / 3], atol=1e-14)


@pytest.mark.parametrize("r", [5.0, 15.0, 28.0])
def test_lorenz_fixed_points_closed_form(r):
    # C+- = (+-sqrt(beta (r-1)), +-sqrt(beta (r-1)), r-1) solve f = 0 (Strogatz, cited at PAPER.md:79).
    b = 8.0 / 3.0
    q = np.sqrt(b * (r - 1))
    for s in (1, -1):
        dx = O.rhs(O.LORENZ, [s * q, s * q, r - 1], [10.0, r, b])
        assert np.max(np.abs(dx)) < 1e-12


def test_lorenz_golden_values():
    g = json.load(open(os.path.join(GOLD, "lorenz_golden.json")))
    for c in g["cases"]:
        p = [g["sigma"], c["r"], g["beta_num"] / g["beta_den"]]
        x = O.rk4(O.LORENZ, np.array(g["x0"])[:, None], p, g["dt"], c["steps"])[:, 0]
        np.testing.assert_allclose(x, c["x"], rtol=g["rtol"], atol=1e-15)


def test_lorenz_r_below_one_collapses_to_origin():
    # PAPER.md:87 "For values of r less than 1, the origin is the only stable fixed point";
    # >= 99% within 1e-2 of the origin at t=50.
    x = O.rk4(O.LORENZ, lorenz_box(2000, 10), [10.0, 0.5, 8 / 3], 0.01, 5000)
    d = np.linalg.norm(x, axis=0)
    assert np.mean(d < 1e-2) >= 0.99


def test_lorenz_r5_two_stable_fixed_points():
    # past the pitchfork at r=1 two new stable fixed points; at r=5 every particle
    # ends at one of C+- (SPEC.md:485).
    r, b = 5.0, 8.0 / 3.0
    q = np.sqrt(b * (r - 1))
    x = O.rk4(O.LORENZ, lorenz_box(500, 11), [10.0, r, b], 0.01, 10000)
    dp = np.linalg.norm(x - np.array([[q], [q], [r - 1]]), axis=0)
    dm = np.linalg.norm(x - np.array([[-q], [-q], [r - 1]]), axis=0)
    assert np.all(np.minimum(dp, dm) < 1e-2)
    assert np.any(dp < 1e-2) and np.any(dm < 1e-2)


def test_lorenz_r28_bounded_attractor():
    # PAPER.md:93 strange attractor; bounded |x|,|y| < 30, 0 < z < 60 over t in [20, 40].
    x = O.rk4(O.LORENZ, lorenz_box(300, 12), LORENZ_P, 0.01, 2000)
    ok = np.ones(x.shape[1], bool)
    for _ in range(20):
        x = O.rk4(O.LORENZ, x, LORENZ_P, 0.01, 100)
        ok &= (np.abs(x[0]) < 30) & (np.abs(x[1]) < 30) & (x[2] > 0) & (x[2] < 60)
    assert ok.mean() >= 0.99


def test_lorenz_spirals_stable_below_hopf_unstable_above():
    # C+- remain stable until r ~ 24.74 (= sigma(sigma+beta+3)/(sigma-beta-1)).
    b = 8.0 / 3.0
    assert 10 * (10 + b + 3) / (10 - b - 1) == pytest.approx(24.74, abs=5e-3)
    for r, stable in ((22.0, True), (27.0, False)):
        q = np.sqrt(b * (r - 1))
        c = np.array([[q], [q], [r - 1]])
        x = O.rk4(O.LORENZ, c + 1e-3, [10.0, r, b], 0.01, 3000)
        d = np.linalg.norm(x - c)
        assert (d < 1e-3) == stable


# ----------------------------------------------------------------------------- HH
HH_DEFAULTS = dict(C=1.0, g_na=120.0, g_k=36.0, g_lk=0.3, e_na=115.0, e_k=-12.0, e_lk=10.613,
                   g_syn=0.5, e_syn=10.0, tau_r=0.5, tau_d=3.0, sigma=5.0, theta=20.0)


def hh_p(n, **kw):
    d = dict(HH_DEFAULTS)
    d.update({f"I{i + 1}": 10.0 for i in range(n)})
    d.update(kw)
    return np.array([d[k] for k in O.hh_param_names(n)])


def test_lorenz_homoclinic_explosion_near_13_9():
    """'At r ~ 13.926 a homoclinic bifurcation occurs ... beyond the bifurcation the
    separatrices have crossed over': below it the origin's outgoing separatrix spirals into the fixed
    point on its own side, above it into the one on the opposite side (the strange
    attractor's appearance at r ~ 13.9 in the bifurcation diagram)."""
    ends = {}
    for r in (13.85, 13.9, 13.95, 14.0):
        p = np.array([10.0, r, 8.0 / 3.0])
        lam = (-11.0 + np.sqrt(81.0 + 40.0 * r)) / 2.0          # unstable eigenvalue of the origin
        v = np.array([1.0, (lam + 10.0) / 10.0, 0.0])
        x = O.rk4(O.LORENZ, (1e-6 * v / np.linalg.norm(v))[:, None], p, 0.001, 200000)
        c = np.sqrt(8.0 / 3.0 * (r - 1.0))
        assert np.abs(np.abs(x[:2, 0]) - c).max() < 1e-6 and abs(x[2, 0] - (r - 1.0)) < 1e-6   # settled on C+-
        ends[r] = np.sign(x[0, 0])
    assert ends[13.85] == ends[13.9] == 1.0 and ends[13.95] == ends[14.0] == -1.0


def _lorenz_lyapunov(r, n=3000, every=10, dt=0.01):
    """Largest Lyapunov exponent (two trajectories, renormalised every `every` steps)."""
    p = np.array([10.0, r, 8.0 / 3.0])
    x = O.rk4(O.LORENZ, np.array([[1.0], [1.0], [20.0]]), p, dt, 5000)
    y = x.copy()
    y[0, 0] += 1e-8
    s = 0.0
    for _ in range(n):
        x = O.rk4(O.LORENZ, x, p, dt, every)
        y = O.rk4(O.LORENZ, y, p, dt, every)
        d = np.linalg.norm(y - x)
        s += np.log(d / 1e-8)
        y = x + (y - x) * (1e-8 / d)
    return s / (n * every * dt)


def test_lorenz_chaos_and_the_periodic_window_near_92():
    """PAPER.md:95, :100 (Fig. 4): 'small windows of parameter values where the dynamics become
    regular ... for example at r = 92': the largest Lyapunov exponent is ~0.91 at r = 28 (textbook 0.906), ~0 inside the
    window (r = 92.5, 93: a stable periodic orbit) and > 1 on both sides of it (r = 90, 95)."""
    assert 0.85 < _lorenz_lyapunov(28.0) < 0.97
    for r in (92.5, 93.0):
        assert abs(_lorenz_lyapunov(r)) < 0.03, r
    for r in (90.0, 95.0):
        assert _lorenz_lyapunov(r) > 1.0, r


def test_hh_gate_steady_states_textbook():
    # Textbook HH gate values at rest (V = 0): m 0.0529, h 0.5961, n 0.3177.
    gold = json.load(open(os.path.join(GOLD, "paper_values.json")))["hh"]["textbook_gates_at_rest"]
    p = hh_p(1, g_syn=0.0, I1=0.0)
    for k, idx in (("h", 1), ("m", 2), ("n", 3)):
        lo, hi = 0.0, 1.0  # bisection on the gate's derivative, which is decreasing in the gate
        for _ in range(60):
            mid = (lo + hi) / 2
            x = [0.0, 0.5, 0.5, 0.5, 0.0]
            x[idx] = mid
            if O.rhs(O.HH, x, p)[idx] > 0:
                lo = mid
            else:
                hi = mid
        assert lo == pytest.approx(gold[k], abs=6e-5)


def test_hh_rest_potential_zero():
    # with I = I_syn = 0 the membrane approaches a fixed point at 0 mV.
    x0 = np.array([[5.0], [0.6], [0.05], [0.32], [0.0]])
    x = O.rk4(O.HH, x0, hh_p(1, g_syn=0.0, I1=0.0), 0.01, 20000)
    assert abs(x[0, 0]) < 0.05


def _count_spikes(x, p, steps, dt=0.01, every=10):
    cnt = np.zeros(x.shape[1])
    times = [[] for _ in range(x.shape[1])]
    prev = x[0].copy()
    for k in range(steps // every):
        x = O.rk4(O.HH, x, p, dt, every)
        up = (prev < 20) & (x[0] >= 20)
        cnt += up
        for i in np.nonzero(up)[0]:
            times[i].append((k + 1) * every * dt)
        prev = x[0].copy()
    return x, cnt, times


def test_hh_onset_of_repetitive_firing_near_6_25():
    # "As I_1 is increased past I_1 ~ 6.25 ... a stable limit cycle appears".
    rng = np.random.default_rng(20)
    n = 128
    x0 = np.vstack([rng.uniform(-20, 100, n), rng.uniform(0, 1, (4, n))])
    counts = {}
    for I in (6.2, 6.3):
        p = hh_p(1, g_syn=0.0, I1=I)
        x = O.rk4(O.HH, x0, p, 0.01, 20000)
        _, cnt, _ = _count_spikes(x, p, 10000)
        counts[I] = cnt
    assert np.all(counts[6.2] == 0)
    assert np.mean(counts[6.3] >= 3) > 0.5


def test_hh_period_at_I10():
    # Repetitive firing at I = 10; period 14.64 ms (SURVEY.md:507, independent
    # computation), inter-spike-interval CV < 5%.
    p = hh_p(1, g_syn=0.0, I1=10.0)
    x = O.rk4(O.HH, np.array([[0.0], [0.596], [0.053], [0.318], [0.0]]), p, 0.01, 10000)
    _, cnt, times = _count_spikes(x, p, 20000, every=1)
    isi = np.diff(times[0])
    assert cnt[0] >= 5
    assert np.mean(isi) == pytest.approx(14.64, abs=0.05)
    assert np.std(isi) / np.mean(isi) < 0.05


def test_hh_ring_index_wraps():
    # PAPER.md:133, reading R9: neuron 1 receives s of neuron N. With only s_N nonzero, only
    # neuron 1's V derivative changes when g_syn changes.
    n = 3
    x = np.array([0.0, 0.6, 0.05, 0.32, 0.0] * n)
    x[5 * (n - 1) + 4] = 0.8
    a = O.rhs(O.HH, x, hh_p(n, g_syn=0.0))
    b = O.rhs(O.HH, x, hh_p(n, g_syn=0.5))
    dv = b[0::5] - a[0::5]
    assert dv[0] == pytest.approx(0.5 * (10.0 - 0.0) * 0.8)
    assert dv[1] == 0 and dv[2] == 0


def test_hh_ring_synchronises():
    # "a very stable synchronous state"; > 50% of random-IC
    # particles synchronous (max pairwise |V_i - V_j| < 5 mV over a period) after t = 500 ms.
    rng = np.random.default_rng(21)
    n = 96
    x0 = np.vstack([np.vstack([rng.uniform(-20, 100, n), rng.uniform(0, 1, (4, n))]) for _ in range(3)])
    p = hh_p(3)
    x = O.rk4(O.HH, x0, p, 0.01, 50000)
    worst = np.zeros(n)
    for _ in range(150):
        x = O.rk4(O.HH, x, p, 0.01, 10)
        V = x[0::5]
        worst = np.maximum(worst, V.max(axis=0) - V.min(axis=0))
    assert np.mean(worst < 5.0) > 0.5


def test_hh_ring_two_spiking_one_silent_cycles():
    """PAPER.md:158 against reading R8's (unpublished) synapse constants: besides the synchronous
    state, random initial conditions settle on three limit cycles where two neurons spike and the
    third is silent -- one per silent neuron -- and in each the pre-synaptic neuron fires first,
    followed by the post-synaptic one, followed by a pause. (PAPER.md:160's small-basin cycle with all
    three firing in the order 1, 3, 2 is not reproduced: with R8's constants the three-neuron
    sequence cycle runs 1, 2, 3, with the coupling -- DESIGN.md R8.)"""
    rng = np.random.default_rng(22)
    n = 256
    x0 = np.vstack([np.vstack([rng.uniform(-20, 100, n), rng.uniform(0, 1, (4, n))]) for _ in range(3)])
    p = hh_p(3)
    x = O.rk4(O.HH, x0, p, 0.01, 40000)                     # 400 ms
    prev = x[0::5].copy()
    times = [[[] for _ in range(n)] for _ in range(3)]
    for k in range(1000):                                    # the next 100 ms, spike = V up through 20 mV
        x = O.rk4(O.HH, x, p, 0.01, 10)
        V = x[0::5]
        for i, j in zip(*np.nonzero((prev < 20) & (V >= 20))):
            times[i][j].append((k + 1) * 0.1)
        prev = V.copy()
    seen = set()
    for j in range(n):
        firing = [len(times[i][j]) >= 4 for i in range(3)]
        silent = [len(times[i][j]) == 0 for i in range(3)]
        if sum(firing) != 2 or sum(silent) != 1:
            continue
        q = silent.index(True)                 # silent neuron; (q+1) receives from q (reading R9)
        pre, post = (q + 1) % 3, (q + 2) % 3   # post receives from pre
        tp, tq = np.array(times[pre][j]), np.array(times[post][j])
        lag = [tq[tq > t][0] - t for t in tp[:-1] if np.any(tq > t)]       # pre -> next post spike
        back = [tp[tp > t][0] - t for t in tq[:-1] if np.any(tp > t)]      # post -> next pre spike
        assert np.mean(lag) < np.mean(back), (j, q)          # pre fires first, then post, then a pause
        seen.add(q)
    assert seen == {0, 1, 2}


# ----------------------------------------------------------------------------- STN-GPe
STN_DEFAULTS = dict(w_ss=0.0, w_gs=8.971, w_sg=15.168, w_gg=8.502, I=2.216, tau_s=1.0, tau_g=2.77,
                    a_s=2.891, theta_s=2.049, a_g=1.826, theta_g=2.032)


def stn_p(**kw):
    d = dict(STN_DEFAULTS)
    d.update(kw)
    return np.array([d[k] for k in O.PARAMS[O.STN]])


def test_stn_uncoupled_closed_form():
    # With w_ss = w_gs = w_sg = w_gg = 0, Eqs. 1-2 become linear:
    # tau x' = -x + Z(const); RK4 gives x_n = x* + (x0 - x*) T4(-h/tau)^n exactly.
    p = stn_p(w_ss=0, w_gs=0, w_sg=0, w_gg=0)
    h, n = 0.01, 300
    x0 = np.array([[0.9], [0.1]])
    x = O.rk4(O.STN, x0, p, h, n)
    xs = expit(STN_DEFAULTS["a_s"] * (STN_DEFAULTS["I"] - STN_DEFAULTS["theta_s"]))
    ys = expit(STN_DEFAULTS["a_g"] * (0 - STN_DEFAULTS["theta_g"]))
    T = lambda z: 1 + z + z * z / 2 + z ** 3 / 6 + z ** 4 / 24
    assert x[0, 0] == pytest.approx(xs + (0.9 - xs) * T(-h / STN_DEFAULTS["tau_s"]) ** n, abs=1e-13)
    assert x[1, 0] == pytest.approx(ys + (0.1 - ys) * T(-h / STN_DEFAULTS["tau_g"]) ** n, abs=1e-13)


def test_stn_time_constants_scale_time():
    # tau multiplies the whole left side (Eqs. 1-2): doubling tau_s, tau_g and h gives the same
    # RK4 iterates (exact in real arithmetic; fp64 rounding only).
    rng = np.random.default_rng(30)
    x0 = rng.uniform(0, 1, (2, 20))
    a = O.rk4(O.STN, x0, stn_p(w_ss=7.8), 0.01, 200)
    b = O.rk4(O.STN, x0, stn_p(w_ss=7.8, tau_s=2.0, tau_g=5.54), 0.02, 200)
    np.testing.assert_allclose(a, b, atol=1e-12)


def test_stn_argument_signs_via_step_sigmoid():
    # With a very steep sigmoid, Z_s(u) -> H(u - theta_s) and Z_g(u) -> H(u - theta_g), so
    # tau x' + x tells which side of threshold w_ss x - w_gs y + I (excitatory STN, inhibitory GPe,
    # PAPER.md:40) and -w_gg y + w_sg x fall.
    p = stn_p(w_ss=2.0, w_gs=3.0, w_sg=4.0, w_gg=5.0, I=1.0, a_s=1e4, theta_s=1.5, a_g=1e4, theta_g=0.5,
              tau_s=1.0, tau_g=1.0)
    def z(x, y):
        d = O.rhs(O.STN, [x, y], p)
        return d[0] + x, d[1] + y
    # u_s = 2x - 3y + 1 ; u_g = 4x - 5y
    zs, zg = z(0.5, 0.1)    # u_s = 1.7 > 1.5 ; u_g = 1.5 > 0.5
    assert zs == pytest.approx(1.0) and zg == pytest.approx(1.0)
    zs, zg = z(0.5, 0.2)    # u_s = 1.4 < 1.5 ; u_g = 1.0 > 0.5
    assert zs == pytest.approx(0.0, abs=1e-12) and zg == pytest.approx(1.0)
    zs, zg = z(0.2, 0.1)    # u_s = 1.1 < 1.5 ; u_g = 0.3 < 0.5
    assert zs == pytest.approx(0.0, abs=1e-12) and zg == pytest.approx(0.0, abs=1e-12)


@pytest.mark.parametrize("w_ss", [0.0, 4.9, 7.8, 11.0])
def test_stn_forward_invariance_of_unit_square(w_ss):
    # activity is in (0,1) and Z in (0,1) makes (0,1)^2 forward-invariant.
    rng = np.random.default_rng(31)
    x = O.rk4(O.STN, rng.uniform(0, 1, (2, 500)), stn_p(w_ss=w_ss), 0.01, 1000)
    assert np.all((x > 0) & (x < 1))


def test_stn_backward_particles_leave():
    # backward particles "move very quickly out of the bounds of the system".
    rng = np.random.default_rng(32)
    x = O.rk4(O.STN, rng.uniform(0, 1, (2, 500)), stn_p(), -0.01, 1000)
    out = np.any((x < 0) | (x > 1), axis=0)
    assert out.mean() > 0.95


def _stn_fixed_points(p):
    """Fixed points of Eqs. 1-2 in the unit square (Newton from a grid) with their Jacobian
    eigenvalues (central differences of the oracle's RHS)."""
    from scipy.optimize import fsolve
    F = lambda z: np.asarray(O.rhs(O.STN, [z[0], z[1]], p))
    out = []
    for a in np.linspace(0.02, 0.98, 13):
        for b in np.linspace(0.02, 0.98, 13):
            z, _, ier, _ = fsolve(F, [a, b], full_output=True)
            if ier == 1 and np.all(np.abs(F(z)) < 1e-11) and np.all((z > 0) & (z < 1)) and \
                    not any(np.allclose(z, q, atol=1e-7) for q, _ in out):
                e = 1e-7
                J = np.array([(F(z + [e, 0]) - F(z - [e, 0])) / (2 * e), (F(z + [0, e]) - F(z - [0, e])) / (2 * e)]).T
                out.append((z, np.linalg.eigvals(J)))
    return out


def _stn_forward_orbits(w_ss, n=300, steps=20000):
    """Per-particle range of x (sampled every 5 steps) over the last 2000 steps of `steps` forward
    RK4 steps (dt = 0.01) from uniform ICs in (0,1)^2."""
    rng = np.random.default_rng(33)
    x = O.rk4(O.STN, rng.uniform(0, 1, (2, n)), stn_p(w_ss=w_ss), 0.01, steps - 2000)
    lo, hi = x.copy(), x.copy()
    for _ in range(400):
        x = O.rk4(O.STN, x, stn_p(w_ss=w_ss), 0.01, 5)
        lo, hi = np.minimum(lo, x), np.maximum(hi, x)
    return hi[0] - lo[0], x


def test_stn_paper_phase_portraits_at_w0_w78_w11():
    """The constants of reading R6 (unpublished in the paper) against the phase portraits the paper
    prints (PAPER.md:47, Fig. 2 caption; :50, :52): w_ss = 0 -- a single, globally stable spiral;
    w_ss = 7.8 -- an unstable spiral and a (globally attracting) stable limit cycle; w_ss = 11 -- an
    unstable node, a saddle and a stable node. (At w_ss = 4.9 the paper also shows a pair of limit
    cycles around the stable spiral; with R6's constants the spiral is stable there but no cycle
    pair appears -- DESIGN.md R6.)"""
    fp = _stn_fixed_points(stn_p(w_ss=0.0))
    assert len(fp) == 1
    ev = fp[0][1]
    assert np.all(ev.real < 0) and np.all(np.abs(ev.imag) > 0.1)            # stable spiral
    amp, x = _stn_forward_orbits(0.0)
    assert amp.max() < 1e-9 and np.abs(x - fp[0][0][:, None]).max() < 1e-9  # every particle reaches it

    fp = _stn_fixed_points(stn_p(w_ss=7.8))
    assert len(fp) == 1
    ev = fp[0][1]
    assert np.all(ev.real > 0) and np.all(np.abs(ev.imag) > 0.1)            # unstable spiral
    amp, _ = _stn_forward_orbits(7.8)
    assert amp.min() > 0.5 and amp.max() - amp.min() < 2e-3                 # one stable cycle for all

    fp = _stn_fixed_points(stn_p(w_ss=11.0))
    assert len(fp) == 3
    kinds = sorted((int(np.sum(e.real > 0)), bool(np.all(np.abs(e.imag) < 1e-12))) for _, e in fp)
    assert kinds == [(0, True), (1, True), (2, True)]    # stable node, saddle, unstable node
    amp, _ = _stn_forward_orbits(11.0)
    assert amp.max() < 1e-6                              # no oscillation left (after the SNIC)


def test_stn_bifurcation_order_along_w_ss():
    """PAPER.md:52 (and Fig. 3 caption): increasing w_ss, the fixed point loses stability in an
    Andronov-Hopf bifurcation, then a saddle-node on the invariant circle leaves a new stable fixed
    point -- the Hopf lies between the paper's w_ss = 4.9 (stable spiral) and 7.8 (unstable spiral),
    the SNIC between 7.8 (a cycle) and 11 (three fixed points), and the period grows as the SNIC
    approaches ("bunching up")."""
    from scipy.optimize import brentq

    def re_max(w):
        fp = _stn_fixed_points(stn_p(w_ss=w))
        assert len(fp) == 1
        return fp[0][1].real.max()
    assert re_max(4.9) < 0 < re_max(7.8)
    w_h = brentq(re_max, 4.9, 7.8, xtol=1e-6)
    assert 4.9 < w_h < 7.8
    n_fp = {w: len(_stn_fixed_points(stn_p(w_ss=w))) for w in (7.8, 9.0, 10.0, 10.5, 11.0)}
    first3 = min(w for w, k in n_fp.items() if k == 3)
    assert all(k == 1 for w, k in n_fp.items() if w < first3) and all(k == 3 for w, k in n_fp.items() if w >= first3)
    assert 7.8 < first3 <= 11.0

    def period(w):   # time between successive upward crossings of the cycle's mean x
        _, x = _stn_forward_orbits(w, n=1, steps=20000)
        p = stn_p(w_ss=w)
        xs, c = [], None
        for _ in range(6000):
            x = O.rk4(O.STN, x, p, 0.01, 1)
            xs.append(x[0, 0])
        xs = np.array(xs)
        m = 0.5 * (xs.min() + xs.max())
        up = np.nonzero((xs[:-1] < m) & (xs[1:] >= m))[0]
        return np.diff(up).mean() * 0.01
    assert period(7.8) < period(9.0) < period(10.0)


# ----------------------------------------------------------------------------- front-end coverage model
def test_funcs_model_closed_form_at_origin():
    # sin(0)cos(0) + tanh(0) - (1+0)^0.75 + 0.1 pi ; sqrt(1) - log(2) + exp(0) + |0| - 0 ; 0
    d = O.rhs(O.FUNCS, [0.0, 0.0, 0.0], [1.3, 0.7])
    np.testing.assert_allclose(d, [-1 + 0.1 * np.pi, 2 - np.log(2.0), 0.0], atol=1e-15)
    d32 = O.rhs(O.FUNCS, [0.0, 0.0, 0.0], [1.3, 0.7], dtype=np.float32)
    np.testing.assert_allclose(d32, d, atol=1e-6)


def test_funcs_model_closed_form_at_nontrivial_points():
    """Three points where every term is non-zero and has a distinct value: a swapped sin / cos, a
    wrong pow exponent, a dropped term or a wrong sign changes the result by far more than rounding.
    The expected values are the model's formulas (fireflies_oracle.c rhs_funcs) evaluated with
    Python's math module in double precision."""
    import math as m
    for (x, y, z), (a, b) in (((0.7, -1.3, 0.4), (1.3, 0.7)), ((-2.1, 0.35, -1.7), (0.5, 2.0)),
                              ((1.9, 2.6, 0.9), (-0.8, 0.1))):
        want = [
            m.sin(a * x) * m.cos(y) + m.tanh(z) - (1 + x * x) ** 0.75 + m.pi * 0.1,
            m.sqrt(1 + y * y) - m.log(2 + m.sin(x)) + m.exp(-b * x * x) + abs(z - x) - y ** 3 / 10,
            min(x, y) - max(y, z) / (1 + m.exp(-(x - z))) + (x + y) / (1 + z * z) + m.tan(0.3 * z) - m.e * 0.05 * z,
        ]
        got = O.rhs(O.FUNCS, [x, y, z], [a, b])
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-14)
        got32 = O.rhs(O.FUNCS, [x, y, z], [a, b], dtype=np.float32)
        np.testing.assert_allclose(got32, want, rtol=2e-6, atol=2e-6)
        # and each term matters: perturbing the point changes every component
        moved = O.rhs(O.FUNCS, [x + 0.01, y - 0.01, z + 0.01], [a, b])
        assert np.all(np.abs(moved - got) > 1e-4)


# ----------------------------------------------------------------------------- HH rate removable singularities
def _hh_rates(V, dtype=np.float64):
    """(alpha_m, alpha_n) at membrane potential V from the oracle's HH RHS: with m = n = 0 the gate
    equations reduce to dm/dt = alpha_m(V), dn/dt = alpha_n(V) (PAPER.md:110-129 gating form)."""
    p = hh_p(1, I=0.0)
    x = np.array([V, 0.5, 0.0, 0.0, 0.0], dtype=dtype)
    d = O.rhs(O.HH, x, p, dtype=dtype)
    return d[2], d[3]


def test_hh_alpha_rates_at_their_removable_singularities():
    # alpha_m(V) = 0.1 (25 - V) / (exp((25 - V)/10) - 1) -> 0.1 * 10 = 1 at V = 25;
    # alpha_n(V) = 0.01 (10 - V) / (exp((10 - V)/10) - 1) -> 0.01 * 10 = 0.1 at V = 10 (limit x/(e^(x/y)-1) -> y)
    am, _ = _hh_rates(25.0)
    _, an = _hh_rates(10.0)
    assert am == 1.0 and abs(an - 0.1) < 1e-17
    am32, _ = _hh_rates(25.0, np.float32)
    _, an32 = _hh_rates(10.0, np.float32)
    # float32: 0.01 is not representable; the limit is fl(fl(0.01) * 10), one rounding from 0.1
    assert am32 == np.float32(1.0) and an32 == np.float32(np.float32(0.01) * np.float32(10.0))


@pytest.mark.parametrize("u", [1e-6, -1e-6, 1e-3, -1e-3, 0.05, -0.05, 0.0999, -0.0999])
def test_hh_vtrap_series_branch_against_expm1(u):
    """For |u| < 0.1 (u = x/y) the oracle uses the series y (1 - u/2 + u^2/12 - u^4/720) (reading R10).
    Against x / expm1(x/y) in float64 its relative error must be the first omitted term, u^6/30240
    (Bernoulli series of u/(e^u - 1)) over the function's value, up to rounding: a wrong coefficient would leave an error of
    order u^2 or u^4 instead."""
    for V0, scale in ((25.0, 0.1), (10.0, 0.01)):
        V = V0 - 10.0 * u
        x = V0 - V
        exact = scale * x / np.expm1(x / 10.0)
        am, an = _hh_rates(V)
        got = am if V0 == 25.0 else an
        rel = abs(got - exact) / exact
        g = u / np.expm1(u)   # exact = scale * 10 * g(u): relative error = (u^6/30240) / g(u)
        assert rel <= u ** 6 / 30240 / g * 1.02 + 4e-16, (u, rel)
        if abs(u) <= 1e-3:
            assert rel <= 1e-12


def test_hh_vtrap_continuous_across_the_branch_switch():
    # both sides of |u| = 0.1 agree with the exact function to the series' truncation error (3.3e-11)
    for V0 in (25.0, 10.0):
        for s in (1, -1):
            vals = []
            for uu in (0.1 - 1e-12, 0.1 + 1e-12):
                V = V0 - 10.0 * s * uu
                a = _hh_rates(V)[0 if V0 == 25.0 else 1]
                vals.append(a)
            assert abs(vals[0] - vals[1]) / abs(vals[1]) < 5e-11
