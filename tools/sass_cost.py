"""Read-weighted FP32 issue cost of the innermost RK4 loop of a generated kernel (model from
tools/ubench/pipes.cu on B200: an FFMA2 / FADD2 / FMUL2 reading at most four 32-bit register operand
words runs at full rate; five words at 101/126, six at 87/126). Usage: python tools/sass_cost.py"""
import collections
import re
import sys
import tempfile

sys.path.insert(0, "tools")
sys.path.insert(0, ".")
from sass_reg3 import loop_sass  # noqa: E402

import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems  # noqa: E402


def cost(body):
    total, n, hist = 0.0, 0, collections.Counter()
    for op, rest in body:
        base = op.split(".")[0]
        if base in ("FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL"):
            reads = sum(2 if "F32x2" in x else 1 for x in rest.split(",")[1:] if re.search(r"\bR\d+", x))
            hist[(base, reads)] += 1
            total += 1.0 if reads <= 4 else (1.25 if reads == 5 else 1.5)
            n += 1
    return n, total, hist


if __name__ == "__main__":
    for name, sy in [("lorenz", systems.lorenz()), ("hh", systems.hh_ring(3)), ("stn", systems.stn_gpe())]:
        with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
            f.write(FF.ff_compile_cubin(sy))
            f.flush()
            n, t, h = cost(loop_sass(f.name, "ff_step_p2_t128"))
            print(f"{name:7s} FP32 instructions {n:4d}  read-weighted cost {t:7.2f}  {sorted(h.items())}")
