"""Shadowed long-horizon parity (protocol P2'): the oracle integrates T steps from the
seeded initial conditions and keeps a checkpoint every K steps; at every checkpoint its state is
uploaded into the GPU context (ff_write_state), the GPU integrates K_a steps -- K_a = the system's
Tier-A horizon from the oracle-only calibration -- and its state must be within Tier A
(every particle e <= 1e-5, scaled) of the oracle's K_a steps from the same checkpoint. Chaotic
amplification never accumulates past K_a, so this exercises the whole attractor (or limit cycle) and
every swept parameter value with the hard tolerance, in the throughput launch (packed kernels, the
pipe-balanced RHS variants). Non-finite rule: a particle must be finite in both or non-finite in both,
except one whose checkpoint state is already beyond 1e30 in magnitude (there the overflow step may
differ by one)."""
import numpy as np
import pytest

import oracle as O
from parity import dim_scales, scaled_error

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems  # noqa: E402

LZ_LO, LZ_HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]   # Fig. 3A box
HH_LO, HH_HI = [-20.0, 0, 0, 0, 0] * 3, [100.0, 1, 1, 1, 1] * 3


def _params(s, model, **over):
    d = {p[0]: p[1] for p in s.params}
    d.update(over)
    names = O.hh_param_names(3) if model == O.HH else [p[0] for p in s.params]
    return np.array([d[k] for k in names], np.float32)


# (name, system factory, oracle model, IC box, direction, parameter overrides, sweep, T, K, K_a,
#  particles, launch): each system in its bench kernel (Lorenz 4 per thread; STN-GPe 256-thread pairs
#  and HH 128-thread pairs with enough tiles for the pipe-balanced RHS variants), ragged tails
CASES = [
    ("lorenz_r28_fwd", systems.lorenz, O.LORENZ, LZ_LO, LZ_HI, 1, {"r": 28.0}, None, 1000, 50, 30, 80077, (4, 128)),
    ("lorenz_r_swept", systems.lorenz, O.LORENZ, LZ_LO, LZ_HI, 1, {}, ("r", 0.0, 200.0), 1000, 50, 10, 80077, (4, 128)),
    ("stn_w0_fwd", systems.stn_gpe, O.STN, [0.0, 0.0], [1.0, 1.0], 1, {"w_ss": 0.0}, None, 1000, 50, 50, 160077, (2, 256)),
    ("stn_w7.8_cycle", systems.stn_gpe, O.STN, [0.0, 0.0], [1.0, 1.0], 1, {"w_ss": 7.8}, None, 1000, 50, 50, 160077,
     (2, 256)),
    ("stn_w0_bwd", systems.stn_gpe, O.STN, [0.0, 0.0], [1.0, 1.0], -1, {"w_ss": 0.0}, None, 1000, 50, 50, 160077,
     (2, 256)),
    ("hh_ring3", lambda: systems.hh_ring(3), O.HH, HH_LO, HH_HI, 1, {}, None, 1000, 50, 10, 80077, (2, 128)),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_shadowed_long_horizon_tier_a(case):
    name, make, model, lo, hi, direction, over, sweep, T, K, K_a, n, launch = case
    s = make()
    p = _params(s, model, **over)
    h = np.float32(0.01 * direction)
    ctx = FF.Context(s, [n])
    ctx.set_launch(*launch)
    for k, v in over.items():
        ctx.set_param(k, v)
    g = ctx.init_group(lo, hi, n, direction, 0, seed=41)
    sv, sidx = None, -1
    if sweep:
        ctx.sweep_param(g, sweep[0], sweep[1], sweep[2], 0, seed=42)
        sv = O.sweep_values(sweep[1], sweep[2], 0, 42, 0, n, n)
        sidx = [q[0] for q in s.params].index(sweep[0])
    sc = dim_scales(lo, hi)
    x = O.ic_uniform(lo, hi, 41, 0, n)
    checked = worst = 0
    for c in range(0, T, K):
        ok = np.all(np.isfinite(x), axis=0) & np.all(np.abs(x) <= 1e30, axis=0)
        ctx.write_state(g, x)
        ctx.step(K_a, 0.01)                            # (the group's direction signs it: h = direction dt)
        got = ctx.read_state(g)
        want = O.rk4(model, x, p, h, K_a, sidx, sv)
        fg, fo = np.all(np.isfinite(got), axis=0), np.all(np.isfinite(want), axis=0)
        assert np.array_equal(fg[ok], fo[ok]), f"{name} step {c}: finite on one side only"
        both = ok & fg & fo
        e = scaled_error(got[:, both], want[:, both], sc)
        if e.size:
            worst = max(worst, float(e.max()))
            assert e.max() <= 1e-5, f"{name}: checkpoint {c}, max e {e.max():.3g}"
        checked += int(both.sum())
        x = O.rk4(model, x, p, h, K, sidx, sv)      # the oracle's own trajectory to the next checkpoint
    assert checked >= (T // K) * n // 2, name          # most particles checked at most checkpoints
    print(f"shadow {name}: {T // K} checkpoints x {K_a} steps, {checked} particle-checks, max e {worst:.3g}")
