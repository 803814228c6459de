"""Diagnose the pitchfork pin (tests/test_gpu_parity.py): swept Lorenz r in [0, 13), 2^20 particles;
GPU state vs the oracle's after the same steps, split into launches of different lengths."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
sys.path.insert(0, '/root/repo/tests')
import oracle as O  # noqa: E402
import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems  # noqa: E402
from parity import dim_scales, scaled_error  # noqa: E402
LZ_LO, LZ_HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]
P = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
n = 1 << 20
m = 20000
sv = O.sweep_values(0.0, 13.0, 0, 32, 0, n, n)
x0 = O.ic_uniform(LZ_LO, LZ_HI, 31, 0, n)[:, :m]
for plan in ([1000, 1000], [2000], [1000, 1000, 1000], [100] * 20):
    ctx = FF.Context(systems.lorenz(), [n])
    ctx.set_param("r", 28.0)
    g = ctx.init_group(LZ_LO, LZ_HI, n, 1, 0, seed=31)
    ctx.sweep_param(g, "r", 0.0, 13.0, 0, seed=32)
    for S in plan:
        ctx.step(S, 0.01)
    x = ctx.read_state(g)
    xo = O.rk4(O.LORENZ, x0, P, np.float32(0.01), sum(plan), 1, sv[:m])
    e = scaled_error(x[:, :m], xo, dim_scales(LZ_LO, LZ_HI)).max(axis=0)
    r = sv.astype(np.float64)
    mid = (r > 1.5) & (r < 12.5)
    c = np.sqrt(8 / 3 * (r[mid] - 1))
    print(plan[:3], len(plan), 'max e %.3g' % e.max(), 'n bad', int((e > 1e-3).sum()), 'first bad', np.nonzero(e > 1e-3)[0][:5],
          'gpu dev all %.3g' % np.abs(np.abs(x[0, mid]) - c).max(), flush=True)
    ctx.close()
