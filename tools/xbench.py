"""Plain vs exchange-bound step launches at several S: event-timed per-launch cost, to separate the
exchange's constant cost from any per-step slowdown. Since world size 1 launches no
exchange kernel, the measured +19-23 us per frame was taken before that change (commit history)."""
import sys

import numpy as np
import torch

import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import dist as ffdist
from paper_1505_00344_b200 import systems, views


def make(fused):
    ctx = FF.Context(systems.lorenz(), [1 << 22, 1 << 22])
    ctx.init_group([-10, -30, 0], [10, 30, 50], 1 << 22, 1, 0, 2)
    ctx.init_group([-10, -30, 0], [10, 30, 50], 1 << 22, -1, 1, 3)
    M = views.look_at((0, -120, 25), (0, 0, 25), (0, 0, 1))
    P = views.perspective(45, 1, 1, 1000)
    mvp = (P @ M).astype(np.float32)
    if fused:
        img = ffdist.bind_exchanged_image(ctx, [0, 1, 2], mvp, 1024, 1024, 2)
    else:
        img = ctx.project([0, 1, 2], mvp, 1024, 1024, 2)
    return ctx, img


def timeit(ctx, img, S, reps):
    flush = torch.ones(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")
    ts = []
    for i in range(reps + 2):
        torch.sum(flush, dim=0, out=sink)
        img.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.step(S, 0.01)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1000)
    ctx.sync()
    return np.median(ts)


if __name__ == "__main__":
    plain, fused = make(False), make(True)
    for S in [int(s) for s in sys.argv[1:]] or [1, 10, 100, 1000]:
        reps = 20 if S < 1000 else 5
        a, b = timeit(*plain, S, reps), timeit(*fused, S, reps)
        print(f"S={S:5d} plain {a:9.1f} us  fused {b:9.1f} us  diff {b - a:7.1f} us", flush=True)
