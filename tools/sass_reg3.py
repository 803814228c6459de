"""Count packed FP32 instructions by operand kind in the innermost RK4 loop of a generated kernel:
FFMA2 with three per-thread register-pair operands runs at ~68% of the FP32 pipe rate on B200
(register-file read bandwidth; tools/ubench/pipes.cu), so the front end avoids them where it can.
Usage: python tools/sass_reg3.py lorenz|hh|stn [kernel]"""
import collections
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, ".")
import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems  # noqa: E402


def loop_sass(cubin, kernel):
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", kernel, cubin], capture_output=True, text=True).stdout
    ins = []
    for ln in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    best = None
    for a, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < a:
                body = [(o, r) for (b, o, r) in ins if int(t.group(1), 16) <= b <= a]
                if sum(o.startswith(("FFMA2", "FFMA")) for o, _ in body) >= 20 and (best is None or len(body) < len(best)):
                    best = body
    return best or []


def classify(body):
    c = collections.Counter()
    for op, rest in body:
        base = op.split(".")[0]
        if base in ("FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL"):
            regs = len(re.findall(r"\bR\d+", rest)) - 1   # minus the destination
            c[f"{base} {regs}reg"] += 1
    return c


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "lorenz"
    kern = sys.argv[2] if len(sys.argv) > 2 else "ff_step_p2_t128"
    sy = {"lorenz": systems.lorenz, "hh": lambda: systems.hh_ring(3), "stn": systems.stn_gpe}[name]()
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(FF.ff_compile_cubin(sy))
        f.flush()
        for k, v in sorted(classify(loop_sass(f.name, kern)).items()):
            print(f"{k:14s} {v}")
