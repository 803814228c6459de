"""Two ranks as two contexts on one GPU (Lorenz configs[1] sharded in halves, 1024^2 x 2 image, each
rank on its own stream): event-timed frame (zero + ff_step on both ranks) with no exchange, with the
sum-pass exchange (ff_set_exchange) and with the push exchange (ff_set_exchange_push), at several S.
On one GPU the "peer" reductions stay in local HBM/L2, so this measures the barriers, the system-scope
REDs and, for push, the doubled REDs -- not NVLink."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems, views  # noqa: E402
from paper_1505_00344_b200.fireflies import ff_set_stream  # noqa: E402

N = 1 << 22


def make(mode):
    world = 2
    streams = [torch.cuda.Stream() for _ in range(world)]
    M = views.look_at((0, -120, 25), (0, 0, 25), (0, 0, 1))
    P = views.perspective(45, 1, 1, 1000)
    mvp = (P @ M).astype(np.float32)
    ranks = []
    for r in range(world):
        ctx = FF.Context(systems.lorenz(), [N, N], rank=r, world=world)
        ff_set_stream(ctx.ctx, streams[r].cuda_stream)
        ctx.stream = streams[r]
        ctx.init_group([-10, -30, 0], [10, 30, 50], N, 1, 0, 2)
        ctx.init_group([-10, -30, 0], [10, 30, 50], N, -1, 1, 3)
        ctx.set_reset(True, None, None, 0.0)
        img = torch.zeros((2, 1024, 1024), dtype=torch.int32, device="cuda")
        ctx.project([0, 1, 2], mvp, 1024, 1024, 2, image=img)
        ctx.set_grid_limit(148 * 4)
        ranks.append((ctx, img))
    sigs = [torch.zeros(8, dtype=torch.int64, device="cuda") for _ in range(world)]
    torch.cuda.synchronize()
    if mode != "plain":
        for r, (ctx, _) in enumerate(ranks):
            ctx.set_exchange(r, world, [i.data_ptr() for _, i in ranks], [s.data_ptr() for s in sigs], 5000.0)
            if mode == "push":
                ctx.set_exchange_push(True)
            ctx._keep_signals = sigs
    return ranks, streams


def timeit(ranks, streams, S, reps):
    flush = torch.ones(64 << 20, device="cuda")
    sink = torch.empty((), device="cuda")
    ts = []
    for i in range(reps + 2):
        torch.sum(flush, dim=0, out=sink)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in streams:
            s.wait_event(e0)
        for (ctx, img), s in zip(ranks, streams):
            with torch.cuda.stream(s):
                img.zero_()
            ctx.step(S, 0.01)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) * 1000)
    for ctx, _ in ranks:
        ctx.sync()
    return float(np.median(ts))


if __name__ == "__main__":
    setups = {m: make(m) for m in ("plain", "sum", "push")}
    for S in [int(s) for s in sys.argv[1:]] or [1, 10, 100]:
        reps = 20
        t = {m: timeit(*setups[m], S, reps) for m in setups}
        print(f"S={S:5d} plain {t['plain']:9.1f} us  sum-pass {t['sum']:9.1f} us ({t['sum'] - t['plain']:+.1f})  "
              f"push {t['push']:9.1f} us ({t['push'] - t['plain']:+.1f})", flush=True)
