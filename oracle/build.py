"""Build the CPU oracle shared library (TEST INFRASTRUCTURE ONLY; see fireflies_oracle.c).

Flags: no FP contraction, no fast-math, so every float operation is one IEEE round-to-nearest
op in source order. OpenMP only parallelises the independent-particle loop.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fireflies_oracle.c")
OUT = os.path.join(HERE, "liboracle.so")
FLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fexcess-precision=standard",
         "-fopenmp", "-shared", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-function"]


def build_timing(out_dir: str) -> str:
    """The same unchanged source built for timing only (bench.py's cpu_baseline.o3_native; SURVEY.md
    8(d) "oracle timing"): -O3 -march=native for the host it runs on, still no FP contraction and no
    fast-math. Timing only (never a parity reference); built on the measuring host, into out_dir."""
    out = os.path.join(out_dir, "liboracle_o3native.so")
    flags = [f if f != "-O2" else "-O3" for f in FLAGS] + ["-march=native"]
    subprocess.run(["gcc", *flags, "-o", out, SRC, "-lm"], check=True)
    return out


def build(force: bool = False) -> str:
    deps = [SRC, os.path.join(HERE, "oracle_impl.h")]
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    cmd = ["gcc", *FLAGS, "-o", OUT + ".tmp", SRC, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
