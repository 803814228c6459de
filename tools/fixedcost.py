"""Per-launch fixed cost decomposition for Lorenz 2^23 particles, no image: event-timed launches at
S = 0 (load only), 1, 2, 4, 8, 16, 32 with the L2 flushed before each launch."""
import numpy as np
import torch

import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import systems

ctx = FF.Context(systems.lorenz(), [1 << 22, 1 << 22])
ctx.init_group([-10, -30, 0], [10, 30, 50], 1 << 22, 1, 0, 2)
ctx.init_group([-10, -30, 0], [10, 30, 50], 1 << 22, 1, 1, 3)
ctx.set_param("r", 0.5)   # bounded trajectories
flush = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")
for S in (0, 1, 2, 4, 8, 16, 32, 100):
    for ppt, tpb in ((2, 128),):
        ctx.set_launch(ppt, tpb)
        ts = []
        for i in range(12):
            torch.sum(flush, dim=0, out=sink)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.step(S, 0.001)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) * 1000)
        print(f"S={S:4d} p{ppt}t{tpb}: {np.median(ts):8.1f} us", flush=True)
