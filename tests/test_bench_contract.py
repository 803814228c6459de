"""bench.py contract checks that run without a GPU: the reference arm (the oracle on the host cores)
prints one JSON line with the driver's keys; the workloads match BASELINE.json's configs."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--config", "stn"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, env=dict(os.environ, FF_BENCH_REF_PARTICLES="65536"))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "stn"


def test_workloads_cover_baseline_configs():
    sys.path.insert(0, ROOT)
    import bench
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert len(base["configs"]) == 5
    w = bench.WORKLOADS
    assert sum(n for n, *_ in w["stn"]["groups"]) == 10000                          # configs[0]
    assert [g[0] for g in w["lorenz3d"]["groups"]] == [1 << 22, 1 << 22]            # configs[1]
    assert w["lorenz3d"]["groups"][1][1] == -1 and w["lorenz3d"]["proj"] == "lorenz_camera"
    assert w["hh"]["groups"][0][0] == 1 << 20 and len(w["hh"]["box"][0]) == 15      # configs[2]
    assert w["sweep"]["groups"][0][0] == 1 << 24 and w["sweep"]["sweep"][1:3] == ("r", 0.0, 200.0)[1:]  # configs[3]
    assert w["lorenz1b"]["groups"][0][0] == 1 << 30 and w["lorenz1b"].get("strong")  # configs[4]


import pytest  # noqa: E402


@pytest.mark.parametrize("config", ["lorenz3d", "sweep", "stn_bif3d", "hh", "lorenz1b", "lorenz3d_collapsed"])
def test_reference_arm_runs_every_workload(config):
    """The oracle sample of every bench workload (swept ones included) runs and prints its line."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--config", config, "--S", "2"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=dict(os.environ, FF_BENCH_REF_PARTICLES="2048"))
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.strip().splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == config


def test_reference_arm_under_torchrun_prints_once():
    """N > 1 (torchrun): rank 0 alone runs the reference arm and prints its line; the other ranks
    exit 0 without work."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "1", "--config", "lorenz3d", "--S", "2"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=dict(os.environ, FF_BENCH_REF_PARTICLES="2048"))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2


def test_frozen_l_alg_matches_the_front_ends_plain_count():
    """L_alg is frozen in bench.py; the front end's plain-formulation count of the same
    RHS text must still agree (STN-GPe, HH ring), Lorenz within the one contraction the survey's probe
    found (45 vs 44)."""
    sys.path.insert(0, ROOT)
    import bench
    for name, (fma, mufu) in bench.L_ALG.items():
        pf, pm, *_ = bench.op_counts(bench.make_system(name), -1)
        assert pm == mufu, name
        assert pf == fma or (name == "lorenz" and pf == fma + 1), (name, pf, fma)
    assert bench.L_ALG["hh_ring3"][1] == 132 and bench.L_ALG["lorenz"] == (44, 0)


def test_gpus_n_without_torchrun_fails_loudly_without_gpus():
    """`bench.py --gpus 2` outside torchrun re-launches itself under torch.distributed.run -- after
    checking that 2 GPUs are visible; here (none) it must exit non-zero with a message, not print a
    1-rank line."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "1", "--config", "stn"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, env=dict(os.environ, CUDA_VISIBLE_DEVICES=""))
    assert out.returncode != 0
    assert "needs 2 visible GPUs" in out.stderr
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_world_size_must_match_gpus():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1",
                          "--warmup", "1", "--config", "stn"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT, env=dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr


def test_paper_context_quotes_table_1():
    """The bench line quotes the paper's Table 1 number for its system, with the
    hardware, as context (vs_baseline stays null: other machine, other particle counts)."""
    import bench
    assert bench.paper_context("lorenz")["particle_steps_per_s"] == 3_000_000 / 3e-3
    assert bench.paper_context("stn_gpe")["particle_steps_per_s"] == 700_000 / 1e-3
    assert bench.paper_context("hh_ring3")["particle_steps_per_s"] == 500_000 / 22e-3
    assert all(bench.paper_context(w["system"]) for w in bench.WORKLOADS.values())


def test_committed_bench_lines_carry_the_contract_keys():
    """The evidence lines under profiles/ (written by bench.py on a B200) carry every key the bench
    contract names: the base line, roofline (bound, achieved, peak, unit, frac, traffic), cpu_baseline
    (value, unit, cores, kind, sample), e2e (value, unit, host<->device bytes), gpu_launches > 0 and
    the clocks sampled under load; the reference arm's line is marked and self-consistent."""
    import json
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    line = json.loads(open(os.path.join(root, "profiles", "r02_bench_default.json")).read().strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["warmup"] >= 3 and line["higher_is_better"] is True
    assert line["config"]["workload"] == "lorenz3d" and "l2" in line["config"]
    r = line["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert 0 < r["frac"] <= 1.0 and r["traffic"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = line["e2e"]
    assert e["unit"] == line["unit"] and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert 0 < e["value"] < line["value"]
    assert line["gpu_launches"] >= line["steps"]
    clk = line["clocks"]
    assert clk["sm_mhz"] > 0 and not set(clk["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    ref = json.loads(open(os.path.join(root, "profiles", "r02_bench_reference.json")).read().strip().splitlines()[-1])
    assert ref["impl"] == "reference" and ref["metric"] == line["metric"] and ref["unit"] == line["unit"]
    assert ref["config"]["workload"] == line["config"]["workload"]
    assert ref["e2e"]["value"] == ref["value"] and ref["cpu_baseline"]["value"] == ref["value"]
