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
