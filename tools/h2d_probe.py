"""Pinned host -> device bandwidth on the box (one 100 MB copy, and 6 x 16.7 MB copies) vs the
e2e frame's ff_write_state path."""
import torch
n = 100663296 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for chunks in (1, 6):
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    for it in range(3):
        s.record()
        for c in range(chunks):
            lo, hi = c * n // chunks, (c + 1) * n // chunks
            d[lo:hi].copy_(h[lo:hi], non_blocking=True)
        e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    print(f"{chunks} chunk(s): {ms:.3f} ms -> {n * 4 / ms / 1e6:.1f} GB/s")
hd = torch.empty(2 * 1024 * 1024, dtype=torch.int32).pin_memory()
dd = torch.empty(2 * 1024 * 1024, dtype=torch.int32, device="cuda")
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record(); hd.copy_(dd, non_blocking=True); e.record(); torch.cuda.synchronize()
print(f"D2H 8 MB: {s.elapsed_time(e):.3f} ms")
