"""Per-launch fixed cost at S = 100 (Lorenz, no image, no reset, r = 0.5 so every trajectory stays
bounded): event-timed launches at 2^23, 2^24 and 2^25 particles, L2 flushed before each. Fixed cost
= 2 t(n) - t(2n); what is left of the FP32 bound is the launch's tail and setup."""
import numpy as np
import torch

import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import systems


def timeit(n_half, S=100, reps=10):
    ctx = FF.Context(systems.lorenz(), [n_half, n_half])
    ctx.init_group([-10, -30, 0], [10, 30, 50], n_half, 1, 0, 2)
    ctx.init_group([-10, -30, 0], [10, 30, 50], n_half, 1, 1, 3)
    ctx.set_param("r", 0.5)
    flush = torch.ones(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")
    ts = []
    for i in range(reps + 2):
        torch.sum(flush, dim=0, out=sink)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.step(S, 0.01)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1000)
    ctx.close()
    return float(np.median(ts))


if __name__ == "__main__":
    t = {n: timeit(n // 2) for n in (1 << 23, 1 << 24, 1 << 25)}
    for n, v in t.items():
        print(f"n = {n:>9d}: {v:8.1f} us  ({n * 100 / (v * 1e-6):.3e} particle-steps/s, "
              f"{n * 100 * 41 / (v * 1e-6) / (148 * 128 * 1.965e9) * 100:.1f}% of the FP32 peak executed)")
    print(f"fixed cost 2 t(2^23) - t(2^24) = {2 * t[1 << 23] - t[1 << 24]:.1f} us; "
          f"2 t(2^24) - t(2^25) = {2 * t[1 << 24] - t[1 << 25]:.1f} us")
