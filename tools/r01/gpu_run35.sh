# Fused exchange diagnostics: phase timestamps (FF_XDEBUG) at S=1 and S=100, world 1.
mkdir -p gpurun_out
cat > /tmp/xd.py <<'PY'
import sys, torch
import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import systems, views, dist as ffdist
import numpy as np
S = int(sys.argv[1])
ctx = FF.Context(systems.lorenz(), [1 << 22, 1 << 22])
ctx.init_group([-10, -30, 0], [10, 30, 50], 1 << 22, 1, 0, 2)
ctx.init_group([-10, -30, 0], [10, 30, 50], 1 << 22, -1, 1, 3)
M = views.look_at((0, -120, 25), (0, 0, 25), (0, 0, 1)); P = views.perspective(45, 1, 1, 1000)
img = ffdist.bind_exchanged_image(ctx, [0, 1, 2], (P @ M).astype(np.float32), 1024, 1024, 2)
for i in range(6):
    img.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.step(S, 0.01); e1.record(); ctx.sync()
    print("event us", 1000 * e0.elapsed_time(e1), file=sys.stderr)
PY
FF_XDEBUG=1 PYTHONPATH=$PWD python /tmp/xd.py 1 2>&1 | tail -4
FF_XDEBUG=1 PYTHONPATH=$PWD python /tmp/xd.py 100 2>&1 | tail -4
