"""GPU parity of a user-defined system exercising every builtin function of the expression grammar
(include/fireflies.h) against the oracle's hand-coded FUNCS model."""
import numpy as np
import pytest

import oracle as O
from parity import dim_scales, tier_a

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200.systems import SystemDef  # noqa: E402

FUNCS = SystemDef("funcs", ["x", "y", "z"], [
    "sin(a*x)*cos(y) + tanh(z) - pow(1 + x^2, 0.75) + pi*0.1",
    "sqrt(1 + y^2) - log(2 + sin(x)) + exp(-b*x^2) + abs(z - x) - y^3/10",
    "min(x, y) - max(y, z)*sigmoid(x - z) + (x + y)/(1 + z^2) + tan(0.3*z) - e*0.05*z",
], [("a", 1.3, None, None), ("b", 0.7, None, None)])


@pytest.mark.parametrize("ppt,tpb", [(1, 256), (2, 256), (4, 128)])
def test_all_builtin_functions(ppt, tpb):
    n, lo, hi = 9000 + 5, [-2.0, -2.0, -1.5], [2.0, 2.0, 1.5]
    ctx = FF.Context(FUNCS, [n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(lo, hi, n, 1, 0, seed=31)
    ctx.step(20, 0.01)
    want = O.rk4(O.FUNCS, O.ic_uniform(lo, hi, 31, 0, n), np.array([1.3, 0.7], np.float32), np.float32(0.01), 20)
    assert tier_a(ctx.read_state(g), want, dim_scales(lo, hi)) <= 1e-5


@pytest.mark.parametrize("ppt,tpb", [(1, 256), (2, 128), (4, 128)])
def test_exponentials_on_the_fma_pipe(monkeypatch, ppt, tpb):
    """Pipe balancing: with FF_TUNE_EXP2P forcing every exponential (exp, sigmoid) of the FUNCS system
    onto the FMA pipe (ff_exp2p: range reduction + degree-5 polynomial), the result still meets Tier A
    against the oracle (libm exp)."""
    monkeypatch.setenv("FF_TUNE_EXP2P", "99")
    n, lo, hi = 9000 + 5, [-2.0, -2.0, -1.5], [2.0, 2.0, 1.5]
    src = FF.ff_emit_source(FUNCS)
    assert "ff_exp2p(" in src and "exponentials on the FMA pipe per particle-step (pipe balancing): 8" in src
    ctx = FF.Context(FUNCS, [n])
    ctx.set_launch(ppt, tpb)
    g = ctx.init_group(lo, hi, n, 1, 0, seed=31)
    ctx.step(20, 0.01)
    want = O.rk4(O.FUNCS, O.ic_uniform(lo, hi, 31, 0, n), np.array([1.3, 0.7], np.float32), np.float32(0.01), 20)
    assert tier_a(ctx.read_state(g), want, dim_scales(lo, hi)) <= 1e-5


def test_exp2p_extreme_arguments():
    """ff_exp2p clamps its argument to [-126, 126]: exp of very negative arguments gives ~0 and of
    very positive ones a huge positive value (the RK4 sum may then overflow to +inf, as with MUFU) --
    never NaN or garbage exponent bits; sigmoid saturates to 0 / 1."""
    import os
    os.environ["FF_TUNE_EXP2P"] = "99"
    try:
        sysd = SystemDef("ext", ["x", "y"], ["exp(x) * 1e-30", "sigmoid(y)"], [])
        n = 512
        ctx = FF.Context(sysd, [n])
        g = ctx.init_group([-500.0, -500.0], [500.0, 500.0], n, 1, 0, seed=3)
        x0 = ctx.read_state(g)
        ctx.step(1, 1e-3)
        got = ctx.read_state(g)
    finally:
        del os.environ["FF_TUNE_EXP2P"]
    assert not np.any(np.isnan(got))
    assert np.all(got[0][x0[0] < -100] == x0[0][x0[0] < -100])    # exp -> ~0: x unchanged
    assert np.all(got[0][x0[0] > 90] > x0[0][x0[0] > 90])          # huge positive (or +inf)
    s = (got[1] - x0[1]).astype(np.float64) / 1e-3
    assert np.all(np.abs(s[x0[1] > 100] - 1) < 0.1) and np.all(np.abs(s[x0[1] < -100]) < 0.1)   # ulp(400) = 3e-5


@pytest.mark.parametrize("stages", ["0", "4"])
def test_pair_reciprocals_on_the_fma_pipe(monkeypatch, stages):
    """Pipe balancing: the two sigmoids of an evaluation share one reciprocal (exponentials clamped at
    2^60), and with FF_TUNE_RCPP_STAGES=4 that reciprocal runs on the FMA pipe in every stage
    (ff_rcpp: bit-trick estimate + 3 Newton steps). u, v are constant, so one RK4 step of size 1 gives
    z = sigmoid(u) + 2 sigmoid(v) exactly up to rounding: checked against float64 over arguments that
    reach both saturations, in the throughput kernel."""
    monkeypatch.setenv("FF_TUNE_RCP_PAIRS", "1")
    monkeypatch.setenv("FF_TUNE_RCPP_STAGES", stages)
    monkeypatch.setenv("FF_TUNE_EXP2P_STEP", "0")
    sysd = SystemDef("pairs", ["u", "v", "z"], ["0", "0", "sigmoid(u) + 2 * sigmoid(v)"], [])
    src = FF.ff_emit_source(sysd)
    assert "sigmoid pairs sharing a reciprocal: 1" in src
    assert f"stages with the pair reciprocals on the FMA pipe: {stages}" in src
    assert ("ff_rcpp(" in src.split("ff_rhs_v0", 1)[1]) == (stages == "4")
    n = 80000 + 3   # enough tiles for the pipe-balanced (throughput) variant
    ctx = FF.Context(sysd, [n])
    g = ctx.init_group([-200.0, -200.0, 0.0], [200.0, 200.0, 1.0], n, 1, 0, seed=5)
    x0 = ctx.read_state(g)
    x0[2] = 0.0
    ctx.write_state(g, x0)
    x0 = x0.astype(np.float64)
    ctx.step(1, 1.0)
    got = ctx.read_state(g)
    sig = lambda a: 0.5 * (1.0 + np.tanh(0.5 * a))   # noqa: E731  (float64, overflow-free)
    want = sig(x0[0]) + 2 * sig(x0[1])
    assert np.isfinite(got).all()
    assert np.abs(got[2] - want).max() <= 1e-6 * 3
    assert (np.abs(got[2] - want) / np.maximum(want, 1e-3)).max() <= 1e-6
