"""SASS checks of the generated kernels (CPU only: NVRTC + cuobjdump): the inner RK4 loop of the
default Lorenz kernel (2 steps per iteration) issues exactly the expected FMA-pipe work, packed, without spills: 41 FP32
lane-ops per particle-step (4 RHS evaluations x 5 -- sigma factored out of dx/dt into the step
constants -- plus 3 dimensions x 7 for the stage inputs and the RK4 combination)."""
import collections
import re
import subprocess

import pytest

import paper_1505_00344_b200 as FF
from paper_1505_00344_b200 import systems


def inner_loops(cubin_path, kernel):
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", kernel, cubin_path], capture_output=True, text=True).stdout
    ins = []
    for ln in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    loops = []
    for a, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < a:
                lo = int(t.group(1), 16)
                loops.append(collections.Counter(o.split(".")[0] for (b, o, _) in ins if lo <= b <= a))
    return loops


@pytest.fixture(scope="module")
def lorenz_cubin(tmp_path_factory):
    p = tmp_path_factory.mktemp("sass") / "lorenz.cubin"
    p.write_bytes(FF.ff_compile_cubin(systems.lorenz()))
    return str(p)


def test_packed_loop_is_41_lane_ops_per_particle_step_no_spills(lorenz_cubin):
    loops = [c for c in inner_loops(lorenz_cubin, "ff_step_p2_t128") if c["FFMA2"] >= 40]
    assert loops, "no packed RK4 loop found"
    main = min(loops, key=lambda c: sum(c.values()))   # innermost = the smallest loop body
    packed = main["FFMA2"] + main["FMUL2"] + main["FADD2"]
    # unrolled x2, two particles per instruction: 2 steps x 2 particles x 41 lane-ops / 2 lanes
    assert packed == 82
    assert main["LDL"] == 0 and main["STL"] == 0
    assert main["FFMA"] == 0 and main["FADD"] == 0 and main["FMUL"] == 0   # nothing left unpacked


def test_long_launch_register_budget_loop(tmp_path, monkeypatch):
    """The long-launch build of the packed kernel (12 blocks/SM, <= 40 registers; the runtime uses it
    for launches of >= 8 steps) keeps the same 82-instruction packed loop (2 steps), without spills."""
    monkeypatch.setenv("FF_TUNE_MINB_P2_T128", "12")
    p = tmp_path / "lorenz12.cubin"
    p.write_bytes(FF.ff_compile_cubin(systems.lorenz()))
    loops = [c for c in inner_loops(str(p), "ff_step_p2_t128") if c["FFMA2"] >= 40]
    main = min(loops, key=lambda c: sum(c.values()))
    assert main["FFMA2"] + main["FMUL2"] + main["FADD2"] == 82
    assert main["LDL"] == 0 and main["STL"] == 0
    res = subprocess.run(["cuobjdump", "-res-usage", str(p)], capture_output=True, text=True).stdout
    regs = re.search(r"Function ff_step_p2_t128:\s+REG:(\d+)", res)
    assert regs and 32 < int(regs.group(1)) <= 40


def test_scalar_loop_is_41_ops(lorenz_cubin):
    loops = [c for c in inner_loops(lorenz_cubin, "ff_step_p1_t256") if c["FFMA"] >= 40]
    main = min(loops, key=lambda c: sum(c.values()))
    assert main["FFMA"] + main["FADD"] + main["FMUL"] == 82 and main["LDL"] == 0


def test_stn_bifurcation_loop_matches_front_end_count(tmp_path):
    """The pipe-balanced STN-GPe kernel (w_ss swept, the bench's bifurcation workload) executes what
    the front end counts and the roofline's generated-work figures report: per particle-step 11 MUFU
    ops (8 EX2 + 3 RCP: the pair reciprocal of one RK4 stage runs on the FMA pipe) and 73 FP32
    lane-ops, without spills."""
    s = systems.stn_gpe()
    w_ss = [q[0] for q in s.params].index("w_ss")
    p = tmp_path / "stn.cubin"
    p.write_bytes(FF.ff_compile_cubin(s, w_ss))
    loops = [c for c in inner_loops(str(p), "ff_step_p2_t128") if c["MUFU"] >= 8]
    assert loops, "no RK4 loop found"
    main = min(loops, key=lambda c: sum(c.values()))
    # one step per iteration, two particles per thread
    assert main["MUFU"] == 2 * 11
    assert 2 * (main["FFMA2"] + main["FMUL2"] + main["FADD2"]) + main["FFMA"] + main["FMUL"] + main["FADD"] == 2 * 73
    assert main["LDL"] == 0 and main["STL"] == 0


def test_front_end_op_counts():
    """Front-end counts per particle-step (4 RHS evaluations + 7 per dimension): the plain
    formulation (the roofline's algorithmic work) and what the kernel executes after the uniform-
    factor and gating-form rewrites (Lorenz: sigma folded into the step constants; HH: a(1-X) - bX
    -> a - (a+b)X for the 12 gating equations)."""
    import bench
    assert bench.op_counts(systems.lorenz(), -1) == (45, 0, 0, 41, 0, 0)
    # HH plain: 11 MUFU ops per neuron and evaluation (7 exponentials + 4 reciprocals) = 132 per
    # particle-step (SURVEY.md:36); executed: exponentials of one rate argument shared (reading R25)
    assert bench.op_counts(systems.hh_ring(3), -1) == (825, 132, 84, 741, 84, 4)
    # STN-GPe is MUFU-bound: its two sigmoids share one reciprocal, and in one of the four RK4 stages
    # that reciprocal runs on the FMA pipe (ff_rcpp)
    assert bench.op_counts(systems.stn_gpe(), -1) == (62, 16, 8, 73, 11, 4)


def test_pipe_balanced_roofline_work():
    """The ALU roofline's work per particle-step: FMA-bound systems keep their FP32 count; a
    MUFU-bound one gets the least time of both pipes with exponentials movable to the FMA pipe,
    sigmoid pairs sharing a reciprocal and shared reciprocals movable to the FMA pipe."""
    import bench
    assert bench.balanced_work(45, 0, 0) == (45.0, 0, "fma")
    assert bench.balanced_work(813, 84, 36, 4) == (813.0, 0, "fma")
    assert bench.balanced_work(825, 132, 84, 4) == (929.0, 8, "fma+xu")   # HH plain: MUFU-bound
    work, k, pipes = bench.balanced_work(62, 16, 8)
    assert (k, pipes) == (4, "fma+xu") and work == 128 * 12 / 16
    work, k, pipes = bench.balanced_work(62, 16, 8, 4)   # pairs, then one reciprocal on the FMA pipe
    assert (k, pipes) == (0, "fma+xu") and work == 128 * 11 / 16
    assert bench.balanced_work(10, 16, 0) == (128.0, 0, "xu")


def test_bench_kernel_p4_loop(tmp_path, monkeypatch):
    """The bench's headline kernel: ff_step_p4_t128 in its long-launch build (8 blocks/SM, <= 64
    registers; the runtime's choice for Lorenz launches of >= 8 steps): the inner loop holds 2 RK4
    steps of 4 particles -- two independent FFMA2 chains -- = 2 x 4 x 41 / 2 = 164 packed FP32
    instructions, nothing unpacked, no spills."""
    monkeypatch.setenv("FF_TUNE_MINB_P4", "8")
    p = tmp_path / "lorenz_p4.cubin"
    p.write_bytes(FF.ff_compile_cubin(systems.lorenz()))
    loops = [c for c in inner_loops(str(p), "ff_step_p4_t128") if c["FFMA2"] >= 80]
    assert loops, "no packed RK4 loop found"
    main = min(loops, key=lambda c: sum(c.values()))
    assert main["FFMA2"] + main["FMUL2"] + main["FADD2"] == 164
    assert main["FFMA"] == 0 and main["FADD"] == 0 and main["FMUL"] == 0
    assert main["LDL"] == 0 and main["STL"] == 0
    res = subprocess.run(["cuobjdump", "-res-usage", str(p)], capture_output=True, text=True).stdout
    m = re.search(r"Function ff_step_p4_t128:\s+REG:(\d+) STACK:(\d+)", res)
    assert m and int(m.group(1)) <= 64 and int(m.group(2)) == 0


@pytest.mark.parametrize("push", [0, 1, 2])
def test_push_exchange_builds(tmp_path, push):
    """The fused (push) exchange's builds of the bench kernel (ff_set_exchange_push; emitted with
    FF_PUSH = push, compiled here with nvcc from the generated source): the RK4 loop is untouched
    (the same 164 packed instructions, no spills, same register budget), and the histogram's
    reductions are gpu-scope REDs into the bound image (0), system-scope REDs to the peers' images
    (1), or multimem.red.add to the multicast address (2: PTX multimem.red, which ptxas lowers to a
    system-scope REDG on the multicast address -- the NVSwitch fans it out)."""
    src = FF.ff_emit_source(systems.lorenz())
    unroll = re.search(r"#define FF_UNROLL (\d+)", src).group(1)
    src = src.replace("#pragma unroll FF_UNROLL", f"#pragma unroll {unroll}")   # (nvcc: literal only)
    src = src.replace("#define FF_KSEL 255", "#define FF_KSEL 5")
    src = src.replace("#define FF_MINB_P4 ", "#define FF_MINB_P4 8 //")
    if push:
        src = f"#define FF_PUSH {push}\n" + src
    cu = tmp_path / "k.cu"
    cu.write_text(src)
    for kind in ("ptx", "cubin"):
        subprocess.run(["nvcc", f"-{kind}", "-gencode", "arch=compute_100a,code=sm_100a", "-w", "-o",
                        str(tmp_path / f"k.{kind}"), str(cu)], check=True, capture_output=True)
    ptx = (tmp_path / "k.ptx").read_text()
    n_mm = ptx.count("multimem.red.relaxed.sys.global.add.u32")
    n_sys = ptx.count("red.relaxed.sys.global.add.u32") - n_mm
    n_gpu = ptx.count("red.relaxed.gpu.global.add.u32")
    assert (n_mm > 0, n_sys > 0, n_gpu > 0) == (push == 2, push == 1, push == 0)
    loops = [c for c in inner_loops(str(tmp_path / "k.cubin"), "ff_step_p4_t128") if c["FFMA2"] >= 80]
    main = min(loops, key=lambda c: sum(c.values()))
    assert main["FFMA2"] + main["FMUL2"] + main["FADD2"] == 164
    assert main["LDL"] == 0 and main["STL"] == 0
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", "ff_step_p4_t128", str(tmp_path / "k.cubin")],
                          capture_output=True, text=True).stdout
    reds = [r for r in re.findall(r"\bREDG?\.\S*", sass) if ".ADD" in r]
    assert reds and all(("SYS" in r) == (push > 0) for r in reds), set(reds)
    res = subprocess.run(["cuobjdump", "-res-usage", str(tmp_path / "k.cubin")], capture_output=True, text=True).stdout
    m = re.search(r"Function ff_step_p4_t128:\s+REG:(\d+) STACK:(\d+)", res)
    assert m and int(m.group(1)) <= 64 and int(m.group(2)) == 0
