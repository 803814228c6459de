"""Per-launch fixed cost vs tile balance: Lorenz without an image at S = 100 and 400 for a particle
count whose tiles divide evenly over the persistent grid (2368 blocks x 14 tiles x 256) and for the
bench's 2^23 (13.84 tiles per block). Fixed cost = t(S) - S * (t(400) - t(100)) / 300."""
import numpy as np
import torch

import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import systems


def timeit(n_half, S, reps=10):
    ctx = FF.Context(systems.lorenz(), [n_half, n_half])
    ctx.init_group([-10, -30, 0], [10, 30, 50], n_half, 1, 0, 2)
    ctx.init_group([-10, -30, 0], [10, 30, 50], n_half, 1, 1, 3)
    ctx.set_param("r", 0.5)                 # bounded trajectories, no reset bookkeeping
    ts = []
    for i in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.step(S, 0.01)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1000)
    ctx.close()
    return float(np.median(ts))


for name, n_half in [("even (2368 x 14 tiles)", 2368 * 14 * 128), ("bench 2^23", 1 << 22)]:
    t100, t400 = timeit(n_half, 100), timeit(n_half, 400)
    per = (t400 - t100) / 300
    print(f"{name:24s} t100 {t100:8.1f} us  t400 {t400:8.1f} us  per-step {per:6.2f} us  fixed {t100 - 100 * per:6.1f} us")
