"""Bench of the Fireflies hot path on B200 (contract: see DESIGN.md "Measurement").

One bench "step" = one frame of the paper's main loop: zero the density image, then
ONE fused launch that advances every particle S RK4 steps in registers and bins it into the image
(ff_step). N=1 default workload = BASELINE.json configs[1]: Lorenz (sigma 10, r 28, beta 8/3),
2^22 forward + 2^22 backward particles from the Fig. 3A box, dt 0.01, 3-D
perspective density image 1024 x 1024 x 2 channels, S = 100 steps per frame.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config lorenz3d|stn|hh|sweep|lorenz1b]
                  [--S steps_per_frame] [--impl ours|reference]

Under torchrun (N > 1) every rank runs the same per-rank workload on its shard (weak scaling) and
the per-frame image is summed over the ranks (the path's one exchange step): by an
NCCL all-reduce inside the frame's events (default, --exchange nccl), or by the library itself --
its exchange kernel over peer memory after each launch (fused; auto = validated on one frame, else
NCCL; nvls = its sum pass through NVSwitch multicast) or the histogram's own reductions sent to every
rank's image (push; nvls-push = as multimem.red through the multicast address); the time is the max
over ranks. --impl reference
times the CPU oracle (the tier's reference arm) on a bounded sample of the same workload.
"""
import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-steps/s per B200 and per box (Lorenz RK4, 15-D neuron); % FP32 peak"
N_SM = 148
FMA_LANES = 128   # FP32 lanes per SM (FFMA2 does not raise it: profiles/r02_ubench_pipes.txt)
XU_LANES = 16     # MUFU results per clock per SM (same microbenchmark)
RED_PEAK = 2.21e11    # L2 reductions / s on 4 M distinct words (tools/ubench/pipes.cu, profiles/r02_ubench_pipes.txt)
# stream + reductions in one kernel (tools/ubench/red_stream.cu, profiles/r02_ubench_red_stream.txt)
L2_STREAM_BPS, L2_RED_RATE, L2_OVERLAP = 5.174e12, 1.64e11, 75.7 / (38.9 + 51.2)

# Algorithmic work per particle-step: FP32 FMA-pipe lane-ops of the plain
# formulation with a*b+c contracted (Lorenz: 4 RHS x 6 + 3 dims x 7 RK4 combination = 45), MUFU ops
# (exp2 / rcp per evaluation x 4), and HBM bytes per launch-particle (state in + out).
WORKLOADS = {
    "lorenz3d": dict(system="lorenz", groups=[(1 << 22, 1, 0, 2), (1 << 22, -1, 1, 3)], params={"r": 28.0},
                     box=([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]), proj="lorenz_camera", W=1024, H=1024, C=2,
                     S=100, dt=0.01, reset=(None, None, 0.0),
                     desc="Lorenz r=28, 4M fwd + 4M bwd, 3-D perspective image 1024x1024x2, non-finite "
                          "particles reset (PAPER.md:42, :204)"),
    "stn": dict(system="stn_gpe", groups=[(5000, 1, 0, 1), (5000, -1, 1, 11)], params={},
                box=([0.0, 0.0], [1.0, 1.0]), proj=([0, 1], [0.0, 1.0, 0.0, 1.0]), W=512, H=512, C=2,
                S=1000, dt=0.01, 
                desc="STN-GPe 5k fwd + 5k bwd, 1000 steps, 2-D image 512x512x2 (configs[0])"),
    "hh": dict(system="hh_ring3", groups=[(1 << 20, 1, 0, 4)], params={},
               box=([-20.0, 0, 0, 0, 0] * 3, [100.0, 1, 1, 1, 1] * 3), proj=([0, 5], [-20.0, 120.0, -20.0, 120.0]),
               W=1024, H=1024, C=1, S=100, dt=0.01,
               desc="HH ring N=3 (15-D), 1M particles, 2-D (V1,V2) image 1024x1024 (configs[2])"),
    "sweep": dict(system="lorenz", groups=[(1 << 24, 1, 0, 5)], params={}, sweep=("r", 0.0, 200.0, 0, 5),
                  box=([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]), proj=([3, 1], [0.0, 200.0, -160.0, 160.0]),
                  W=2048, H=1024, C=1, S=100, dt=0.01,
                  desc="Lorenz r swept in [0,200), 16M particles, (r, y) image 2048x1024 (configs[3])"),
    "lorenz3d_collapsed": dict(system="lorenz", groups=[(1 << 22, 1, 0, 2), (1 << 22, 1, 1, 3)], params={"r": 0.5},
                               box=([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]), proj="lorenz_camera", W=1024, H=1024,
                               C=2, S=100, dt=0.01, prerun=4000,
                               desc="Lorenz r=0.5 after 4000 steps: 8M particles in ~1 pixel (histogram stress)"),
    "stn_bif3d": dict(system="stn_gpe", groups=[(1 << 22, 1, 0, 21), (1 << 22, -1, 1, 22)], params={},
                      sweep=("w_ss", 0.0, 12.0, 0, 23), reset=([0.0, 0.0], [1.0, 1.0], 0.0),
                      box=([0.0, 0.0], [1.0, 1.0]), proj="stn_box_camera", W=1024, H=1024, C=2, S=100, dt=0.01,
                      
                      desc="STN-GPe 3-D bifurcation (x, y, w_ss in [0,12)), 4M fwd + 4M bwd with reset "
                           "(PAPER.md:54, :59; NEXT row 4)"),
    "lorenz1b": dict(system="lorenz", groups=[(1 << 30, 1, 0, 6)], params={"r": 28.0}, strong=True,
                     box=([-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]), proj="lorenz_camera", W=1024, H=1024, C=1,
                     S=100, dt=0.01, reset=(None, None, 0.0),
                     desc="Lorenz 1B particles sharded over the GPUs (configs[4]), non-finite particles reset"),
}


# The paper's own numbers for this path (Table 1: one RK4 step per particle, averaged
# over 1000 steps, rendering excluded, FP32, GTX 460 / OpenCL): context for the bench line, not the
# target (another machine, other particle counts) -- vs_baseline stays null.
PAPER_TABLE1 = {
    "lorenz": dict(particles=3_000_000, ms_per_step=3.0, cite="PAPER.md:175"),
    "stn_gpe": dict(particles=700_000, ms_per_step=1.0, cite="PAPER.md:174"),
    "hh_ring3": dict(particles=500_000, ms_per_step=22.0, cite="PAPER.md:176"),
}


def paper_context(system):
    t = PAPER_TABLE1.get(system)
    if t is None:
        return None
    return {"hardware": "NVIDIA GeForce GTX 460 (Fermi), OpenCL, FP32 (PAPER.md:178, :225)",
            "particles": t["particles"], "ms_per_step": t["ms_per_step"],
            "particle_steps_per_s": t["particles"] / (t["ms_per_step"] * 1e-3),
            "fps_budget": "30 frames/s incl. rendering (PAPER.md:182)", "source": t["cite"]}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.stop_ev, self.max_mhz = [], set(), threading.Event(), None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x40: "sw_thermal_slowdown",
                 0x80: "hw_thermal_slowdown", 0x100: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_system(name):
    from paper_1505_00344_b200 import systems
    return {"lorenz": systems.lorenz, "stn_gpe": systems.stn_gpe, "hh_ring3": lambda: systems.hh_ring(3)}[name]()


def projection(w):
    from paper_1505_00344_b200 import views
    if w["proj"] == "lorenz_camera":
        return [0, 1, 2], views.lorenz_camera()
    if w["proj"] == "stn_box_camera":
        return [0, 1, 2], views.box_camera([0.0, 0.0, 0.0], [1.0, 1.0, 12.0])
    return w["proj"]


def setup(args, w, rank, world):
    """One context holding the workload's groups (this rank's shard) on torch's current stream, with
    its image bound; returns (ctx, group ids, image, fused)."""
    import torch
    import paper_1505_00344_b200 as FF
    strong = w.get("strong", False)
    # weak scaling: every rank holds the full per-rank workload (global groups = world x per-rank)
    gsizes = [n if strong else n * world for (n, _, _, _) in w["groups"]]
    ctx = FF.Context(make_system(w["system"]), gsizes, rank=rank, world=world)
    for k, v in w["params"].items():
        ctx.set_param(k, v)
    if args.ppt or args.tpb:
        ctx.set_launch(args.ppt, args.tpb)
    lo, hi = w["box"]
    gids = []
    for (n, d, colour, seed), ng in zip(w["groups"], gsizes):
        gids.append(ctx.init_group(lo, hi, ng, d, colour, seed))
    if "sweep" in w:
        name, a, b, mode, seed = w["sweep"]
        for g in gids:
            ctx.sweep_param(g, name, a, b, mode, seed)
    if "reset" in w and not args.no_reset:
        ctx.set_reset(True, *w["reset"])
    if w.get("prerun"):
        ctx.step(w["prerun"], w["dt"])
    axes, view = projection(w)
    fused = not args.no_image and (args.exchange in ("fused", "push") or
                                   (args.exchange in ("auto", "nvls", "nvls-push") and world > 1))
    img = None
    if fused:   # the image sum over ranks is done by the library after each launch, no NCCL call
        from paper_1505_00344_b200 import dist as ffdist
        try:
            # nvls: NVSwitch multicast (torch symmetric memory); push: the histogram's reductions go to
            # every rank's image (ff_set_exchange_push) instead of a sum pass after the launch
            mc = args.exchange in ("nvls", "nvls-push")
            img = ffdist.bind_exchanged_image(ctx, axes, view, w["W"], w["H"], w["C"],
                                              mapping="symmetric" if mc else "auto", multicast=mc,
                                              push=args.exchange in ("push", "nvls-push"))
            if args.exchange in ("auto", "nvls", "nvls-push"):
                ok, why = validate_exchange(ctx, img, w)
                if not ok:
                    raise RuntimeError(why)
        except Exception as e:   # auto: fall back to the NCCL all-reduce, say why in the line
            if args.exchange in ("fused", "push"):
                raise
            args.exchange_note = f"library exchange ({args.exchange}) unavailable ({str(e)[:160]}); NCCL all-reduce used"
            ctx.set_exchange(0, 0)
            fused, img = False, None
    if img is None:
        img = ctx.project(axes, view, w["W"], w["H"], w["C"])
    if args.no_image:   # integration only (HBM roofline of single-step launches without binning)
        ctx.unbind_image()
    torch.cuda.synchronize()
    return ctx, gids, img, fused


def validate_exchange(ctx, img, w):
    """One bin-only frame through the library exchange: it must complete (ff_sync) and leave the same
    image on every rank (checksums compared with MIN / MAX all-reduces)."""
    import torch
    img.zero_()
    ctx.step(0, w["dt"])
    try:
        ctx.sync()
    except Exception as e:
        return False, f"exchange frame failed: {e}"
    v = img.to(torch.float64).flatten()
    wts = torch.arange(1, v.numel() + 1, dtype=torch.float64, device=v.device) % 1009
    ck = torch.stack([v.sum(), (v * wts).sum()])
    lo, hi = ck.clone(), ck.clone()
    torch.distributed.all_reduce(lo, op=torch.distributed.ReduceOp.MIN)
    torch.distributed.all_reduce(hi, op=torch.distributed.ReduceOp.MAX)
    if not torch.equal(lo, hi) or float(lo[0]) <= 0:
        return False, "ranks' exchanged images differ"
    img.zero_()
    return True, ""


def run_ours(args, w, rank, world, device):
    import torch
    S = args.S or w["S"]
    ctx, gids, img, fused = setup(args, w, rank, world)
    n_local = sum(ctx.group_info(g)[1] for g in gids)
    stream = ctx.stream
    # L2 flush = READ 256 MiB (> 126 MB L2) so the cache is refilled with clean lines: a memset would
    # leave ~126 MB of dirty lines whose write-back the next timed kernel would pay for
    flush = torch.ones(64 << 20, dtype=torch.float32, device=device)
    flush_sink = torch.empty((), dtype=torch.float32, device=device)
    dist = world > 1
    reduce = dist and not fused

    def frame():
        if not args.no_image:   # (integration-only frames have no image to clear)
            img.zero_()
        ctx.step(S, w["dt"])
        if reduce:
            torch.distributed.all_reduce(img)

    for _ in range(args.warmup):
        frame()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    if dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(device.index) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            if args.flush == "read":
                torch.sum(flush, dim=0, out=flush_sink)    # L2 flush between timed iterations (not timed)
            elif args.flush == "memset":
                flush.zero_()
            ev[i][0].record(stream)
            if not args.no_image:
                img.zero_()
            ev[i][1].record(stream)
            ctx.step(S, w["dt"])
            if reduce:   # the image sum is part of the frame: it ends before the frame's end event
                torch.distributed.all_reduce(img)
            ev[i][2].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    if dist:
        torch.distributed.barrier()
    launches = ctx.launch_count() - launches0
    frame_ms = np.array([ev[i][0].elapsed_time(ev[i][2]) for i in range(args.steps)])
    kern_ms = np.array([ev[i][1].elapsed_time(ev[i][2]) for i in range(args.steps)])
    t_total = float(frame_ms.sum())
    if dist:
        t = torch.tensor([t_total, float(kern_ms.mean())], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_total, kern_mean = float(t[0]), float(t[1])
        nt = torch.tensor([n_local], dtype=torch.float64, device=device)
        torch.distributed.all_reduce(nt)
        n_total = int(nt.item())
    else:
        kern_mean = float(kern_ms.mean())
        n_total = n_local

    # End-to-end through the C ABI with host buffers, every frame: the whole state from pinned host
    # memory (ff_write_state_async), ff_step, (N > 1: the image sum), the image to pinned host memory
    # (ff_read_image_async). Two contexts on two streams alternate frames, so frame f's copy-in runs
    # while frame f-1 integrates and frame f-2's image is copied out (the copy engines of both
    # directions and the SMs overlap; bytes per frame unchanged). The timed region ends when both
    # streams have finished every frame.
    e2e = None
    if not args.no_e2e:
        from paper_1505_00344_b200 import fireflies as F
        s2 = torch.cuda.Stream(device)
        with torch.cuda.stream(s2):
            ctx2, gids2, img2, _ = setup(args, w, rank, world)
        pair = [(ctx, gids, img, ctx.stream), (ctx2, gids2, img2, s2)]
        host_in = [torch.from_numpy(ctx.read_state(g)).pin_memory() for g in gids]
        host_img = [torch.empty(tuple(img.shape), dtype=torch.int32).pin_memory() for _ in range(2)]
        h2d = sum(t.numel() * 4 for t in host_in)
        d2h = host_img[0].numel() * 4

        def frame_e2e(f):
            c, gs, im, st = pair[f % 2]
            for g, t in zip(gs, host_in):
                F.ff_write_state_async(c.ctx, g, 0, t.shape[1], t.data_ptr())
            with torch.cuda.stream(st):
                im.zero_()
                c.step(S, w["dt"])
                if reduce:
                    torch.distributed.all_reduce(im)
            F.ff_read_image_async(c.ctx, host_img[f % 2].data_ptr())

        for f in range(4):
            frame_e2e(f)
        ke = max(4, min(args.steps, 20))
        torch.cuda.synchronize()
        if dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1, done2 = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                         torch.cuda.Event())
        e0.record(ctx.stream)
        s2.wait_event(e0)
        for f in range(ke):
            frame_e2e(f)
        done2.record(s2)
        ctx.stream.wait_event(done2)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ctx.sync()
        ctx2.sync()
        ms = e0.elapsed_time(e1) / ke
        if dist:
            t = torch.tensor([ms], dtype=torch.float64, device=device)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        e2e = {"value": n_total * S / (ms * 1e-3), "unit": "particle-steps/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ms,
               "path": "per frame: ff_write_state_async (pinned host -> device, whole state), ff_step, "
                       + ("NCCL image all-reduce, " if reduce else "") + "ff_read_image_async (device -> "
                       "pinned host); two contexts on two streams alternate frames so copy-in, integration "
                       "and copy-out of consecutive frames overlap"}
        ctx2.close()
    im_sum = 0 if args.no_image else int(img.sum().item())   # (no image bound: nothing binned)
    ctx.close()
    sweep_idx = -1
    if "sweep" in w:
        sweep_idx = [p[0] for p in make_system(w["system"]).params].index(w["sweep"][0])
    return dict(S=S, n_total=n_total, n_local=n_local, sweep_idx=sweep_idx, t_total_ms=t_total, kern_ms=kern_mean,
                frame_ms=frame_ms, launches=launches, clocks=clk.summary(), e2e=e2e, image_sum=im_sum, fused=fused,
                t_wall=t_wall)


EXP2P_OPS = 8   # FMA-pipe ops of one exponential computed on the FMA pipe (ff_exp2p in ff_device.cuh)
PAIR_OPS = 3    # FMA-pipe ops that let two sigmoids share one reciprocal (one MUFU.RCP fewer)
RCPP_OPS = 7    # FMA-pipe ops of a pair reciprocal computed on the FMA pipe (ff_rcpp in ff_device.cuh)


# L_alg, frozen per system: (FP32 FMA-pipe lane-ops, MUFU ops) per particle-step of
# the plain formulation, a*b+c counted once. Lorenz: 44, the survey's probe of the straight-line RK4
# (216 FFMA + 80 FADD + 58 FMUL per 8 steps; the front end's plain lowering counts 45, one contraction
# fewer). STN-GPe and HH ring (N = 3): the front end's plain count of the RHS as written (no gating
# rewrite, uniform factors multiplied in every evaluation, every exponential and reciprocal on MUFU,
# no exponential sharing), frozen here; tests/test_bench_contract.py checks the front end still
# agrees. HH: 825 + 132 MUFU (11 exponentials per neuron and evaluation, SURVEY.md:36).
L_ALG = {"lorenz": (44, 0), "stn_gpe": (62, 16), "hh_ring3": (825, 132)}


def op_counts(sysdef, sweep_idx):
    """Work per particle-step: (algorithmic FMA-pipe lane-ops, algorithmic MUFU ops, exponentials,
    generated FMA-pipe lane-ops, generated MUFU ops, sigmoid pairs).

    Algorithmic = the plain formulation of the system (as written: no gating-form rewrite, every
    uniform factor of dx/dt multiplied in each of the 4 evaluations, every exponential on MUFU) + the
    RK4 combination (7 per dimension): a fixed per-system constant, so work the front
    end saves raises the fraction instead of shrinking the denominator. Generated = the front end's
    count of what the kernel actually executes."""
    import re
    import paper_1505_00344_b200 as FF
    src = FF.ff_emit_source(sysdef, sweep_idx)
    m = re.search(r"per particle-step, 4 evaluations \(front-end count\): (\d+) arithmetic ops, (\d+) MUFU ops", src)
    p = re.search(r"plain formulation \(no gating rewrite, uniform factors multiplied in every evaluation, no exponential sharing\): "
                  r"(\d+) arithmetic ops, (\d+) MUFU ops, (\d+) exponentials, (\d+) sigmoid pairs", src)
    return (4 * int(p.group(1)) + 7 * sysdef.dim, 4 * int(p.group(2)), 4 * int(p.group(3)),
            int(m.group(1)) + 7 * sysdef.dim, int(m.group(2)), 4 * int(p.group(4)))


def balanced_work(fma_ops, mufu_ops, n_exp, n_pairs=0):
    """FP32-pipe-equivalent work per particle-step of the pipe-balanced roofline: the FMA and MUFU
    pipes run concurrently (128 and 16 results / clk / SM); any exponential can move from MUFU to the
    FMA pipe at EXP2P_OPS ops, two sigmoids can share one reciprocal for PAIR_OPS ops, and r of those
    shared reciprocals can run on the FMA pipe at RCPP_OPS ops, so the least time per particle-step on
    one SM is T = min over k, pairing, r of max((mufu - pairs - k - r) / 16,
    (fma + PAIR_OPS pairs + EXP2P_OPS k + RCPP_OPS r) / 128) cycles; work = 128 T lane-ops (= fma
    for an FMA-bound system). Returns (work, k, binding pipes)."""
    best = (max(mufu_ops / XU_LANES, fma_ops / FMA_LANES), 0, 0)
    for pr in ((0, n_pairs) if n_pairs else (0,)):
        for k in range(0, n_exp + 1):
            for r in range(0, pr + 1):
                t = max((mufu_ops - pr - k - r) / XU_LANES,
                        (fma_ops + PAIR_OPS * pr + EXP2P_OPS * k + RCPP_OPS * r) / FMA_LANES)
                if t < best[0] - 1e-12:
                    best = (t, k, pr or r)
    t, k, pr = best
    moved = k or pr
    pipes = "fma" if fma_ops / FMA_LANES >= mufu_ops / XU_LANES and not moved else ("xu" if not moved else "fma+xu")
    return FMA_LANES * t, k, pipes


def cpu_oracle_sample(w, n_sample, S):
    """Time the oracle (as it stands) on n_sample particles of the workload x S steps + binning."""
    import oracle as O
    model = {"lorenz": O.LORENZ, "stn_gpe": O.STN, "hh_ring3": O.HH}[w["system"]]
    sysdef = make_system(w["system"])
    pvals = {p[0]: p[1] for p in sysdef.params}
    pvals.update(w["params"])
    if model == O.HH:
        names = O.hh_param_names(3)
    else:
        names = O.PARAMS[model]
    p = np.array([pvals[k] for k in names], np.float32)
    lo, hi = w["box"]
    if "sweep" in w:   # swept values exist for the group's own particles only
        n_sample = min(n_sample, w["groups"][0][0])
    x = O.ic_uniform(lo, hi, w["groups"][0][3], 0, n_sample)
    sweep_idx, sv = -1, None
    if "sweep" in w:
        name, a, b, mode, seed = w["sweep"]
        sweep_idx = names.index(name)
        sv = O.sweep_values(a, b, mode, seed, 0, n_sample, w["groups"][0][0])
    axes, view = projection(w)
    t0 = time.perf_counter()
    x = O.rk4(model, x, p, np.float32(w["dt"]), S, sweep_idx, sv)
    O.histogram(x, axes, view, w["W"], w["H"], w["C"], 0, sweep_vals=sv)
    dt = time.perf_counter() - t0
    threads = int(os.environ.get("OMP_NUM_THREADS", 0)) or len(os.sched_getaffinity(0))
    return n_sample * S / dt, dt, threads, n_sample


def host_cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def single_core_oracle(config, n, S):
    """The oracle on ONE host core (OMP_NUM_THREADS=1 in a child process): the analogue of the paper's
    Table 1 "Single Core" column (i5-2500K, gcc -Ofast)."""
    import subprocess
    code = ("import sys; sys.argv=['bench']; import bench; "
            f"v, dt, t, n = bench.cpu_oracle_sample(bench.WORKLOADS[{config!r}], {int(n)}, {int(S)}); "
            "print(v, dt, n)")
    try:
        out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300,
                             env=dict(os.environ, OMP_NUM_THREADS="1"))
        v, dt, n = out.stdout.split()
        return {"value": float(v), "unit": "particle-steps/s", "cores": 1,
                "sample": f"{int(n)} particles x {S} RK4 steps + binning ({float(dt):.1f} s)"}
    except Exception as e:   # the baseline is context; never fail the bench line over it
        return {"error": str(e)[:200]}


def o3_native_oracle(config, n, S):
    """The same oracle source built -O3 -march=native on this host (oracle/build.py build_timing;
    SURVEY.md 8(d) "oracle timing"), all cores, in a child process: how much of the GPU/CPU ratio is
    compiler flags. Context only."""
    import subprocess
    import tempfile
    from oracle import build as obuild
    code = ("import sys; sys.argv=['bench']; import bench; "
            f"bench.cpu_oracle_sample(bench.WORKLOADS[{config!r}], {max(256, int(n) // 16)}, {int(S)}); "   # warm-up
            f"v, dt, t, n = bench.cpu_oracle_sample(bench.WORKLOADS[{config!r}], {int(n)}, {int(S)}); "
            "print(v, dt, t, n)")
    try:
        with tempfile.TemporaryDirectory() as d:
            lib = obuild.build_timing(d)
            out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300,
                                 env=dict(os.environ, FF_ORACLE_LIB=lib))
            v, dt, t, n = out.stdout.split()
        return {"value": float(v), "unit": "particle-steps/s", "cores": int(t),
                "sample": f"{int(n)} particles x {S} RK4 steps + binning ({float(dt):.1f} s)",
                "build": "same source, gcc -O3 -march=native -ffp-contract=off, OpenMP"}
    except Exception as e:   # context only; never fail the bench line over it
        return {"error": str(e)[:200]}


def reference_sample_size(w, S):
    # bounded sample: ~5-12 s of the oracle on a 16-core host (Lorenz ~5e8, STN-GPe ~1.4e8, HH ring
    # ~3.6e7 particle-steps/s measured), i.e. several frames' worth of the workload's particles
    per = {"lorenz": 1 << 25, "stn_gpe": 1 << 24, "hh_ring3": 1 << 21}[w["system"]]
    if os.environ.get("FF_BENCH_REF_PARTICLES"):   # (contract tests on a small CPU)
        return int(os.environ["FF_BENCH_REF_PARTICLES"])
    return max(1024, int(per * 100 / S))


def relaunch(n):
    """`python bench.py --gpus N` without torchrun: re-run this command under torch.distributed.run,
    one rank per GPU on 127.0.0.1 (the driver's own launch), after checking N GPUs are visible.
    Returns torchrun's exit code."""
    import socket
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
        return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="lorenz3d", choices=sorted(WORKLOADS))
    ap.add_argument("--S", type=int, default=0, help="RK4 steps per frame (default per config)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ppt", type=int, default=0)
    ap.add_argument("--tpb", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-image", action="store_true", help="do not bind the image (integration only)")
    ap.add_argument("--flush", default="read", choices=["read", "memset", "none"],
                    help="L2 flush between timed frames (default: read 256 MiB; 'none' only for experiments)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reset", action="store_true", help="(experiments) leave the workload's reset rule off")
    ap.add_argument("--exchange", default="nccl", choices=["auto", "nccl", "fused", "nvls", "push", "nvls-push"],
                    help="per-frame image sum over ranks (N > 1): an NCCL all-reduce (default), or the "
                         "library's exchange over peer memory after each launch (ff_set_exchange; 'auto' "
                         "validates it once and falls back to NCCL) -- not the default until it has run "
                         "across physical GPUs; 'nvls' = the library exchange with its sum pass through "
                         "NVSwitch multicast (multimem), validated likewise; 'push' = the fused exchange "
                         "(ff_set_exchange_push: the histogram's reductions sent to every rank's image over "
                         "peer memory, no sum pass), 'nvls-push' = the same as multimem.red through the "
                         "multicast address, validated with NCCL fallback")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    w = WORKLOADS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        sys.exit(relaunch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world != args.gpus and os.environ.get("FF_BENCH_ONE_DEVICE") != "1":
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    S = args.S or w["S"]
    config = {"workload": args.config, "description": w["desc"], "steps_per_frame": S, "dt": w["dt"],
              "particles_per_gpu": (sum(g[0] for g in w["groups"]) // (world if w.get("strong") else 1)),
              "image": [w["C"], w["H"], w["W"]], "l2": "flushed between timed frames (256 MiB read, outside the timed events)",
              "parallelism": "1 GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        n = reference_sample_size(w, S)
        vals, threads = [], 1
        for _ in range(args.warmup if args.warmup < 3 else 1):
            cpu_oracle_sample(w, max(256, n // 16), S)
        for _ in range(args.steps if args.steps <= 5 else 5):
            v, dt, threads, n = cpu_oracle_sample(w, n, S)
            vals.append(v)
        v = float(np.median(vals))
        sample = f"{n} particles of the workload x {S} RK4 steps + binning per step (oracle, FP32, OpenMP)"
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "particle-steps/s", "n_gpus": args.gpus,
                "steps": len(vals), "warmup": args.warmup, "ms_per_step": n * S / v * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": config,
                "cpu_baseline": {"value": v, "unit": "particle-steps/s", "cores": threads, "kind": "oracle",
                                 "sample": sample, "build": "scalar oracle, gcc -O2 -ffp-contract=off, OpenMP "
                                                             "over particles, no SIMD (not a tuned CPU code)"},
                "e2e": {"value": v, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    # FF_BENCH_DIST_BACKEND=gloo with FF_BENCH_ONE_DEVICE=1: every rank on cuda:0 -- exercises the
    # N > 1 code path on a one-GPU box (plumbing check only; its timings mean nothing)
    backend = os.environ.get("FF_BENCH_DIST_BACKEND", "nccl")
    if os.environ.get("FF_BENCH_ONE_DEVICE") == "1":
        local_rank = 0
    if world > 1:
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group(backend)
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    if world > 1:   # one line per rank on stderr: which GPU each rank drives (stdout holds the JSON line)
        nccl = ".".join(map(str, torch.cuda.nccl.version())) if backend == "nccl" else "-"
        print(f"bench.py: rank {rank}/{world} on cuda:{local_rank} ({torch.cuda.get_device_name(device)}, "
              f"{backend}, NCCL {nccl})", file=sys.stderr, flush=True)
    r = run_ours(args, w, rank, world, device)
    if world > 1:
        how = {"nvls": "image sum by the library's exchange kernel (NVLS multimem sum pass) after each launch",
               "push": "image sum by the histogram itself: its reductions go to every rank's image over NVLink "
                       "peer memory (ff_set_exchange_push), a barrier before and after each launch",
               "nvls-push": "image sum by the histogram itself: its reductions go once each to the images' NVLS "
                            "multicast address (multimem.red), a barrier before and after each launch"}
        config["parallelism"] = f"particles sharded over {world} GPU(s), " + (
            how.get(args.exchange, "image sum by the library's exchange kernel over NVLink peer memory after each launch")
            if r["fused"] else "NCCL image all-reduce per frame")
        config["exchange"] = ({"nvls": "library-nvls", "push": "library-push", "nvls-push": "library-nvls-push"}
                              .get(args.exchange, "library") if r["fused"] else "nccl")
        if getattr(args, "exchange_note", None):
            config["exchange_note"] = args.exchange_note
    if world > 1:
        torch.distributed.destroy_process_group()
    if rank != 0:
        return
    peaks = load_peaks()
    psteps = r["n_total"] * r["S"] * args.steps
    value = psteps / (r["t_total_ms"] * 1e-3)
    clocks = r["clocks"]
    f_max = (peaks.get("sm_max_mhz") or clocks.get("sm_max_mhz") or 1965.0) * 1e6
    kern_s = r["kern_ms"] * 1e-3
    per_launch = r["n_local"] * r["S"]
    # Algorithmic work per particle-step: the plain formulation's FMA-pipe ops (4 RHS evaluations) plus
    # the RK4 combination (7 per dimension) and its MUFU ops; Lorenz: 4 x 6 + 3 x 7 = 45 (the kernel
    # executes 41). The ALU roofline is pipe-balanced (balanced_work): FMA-bound systems report against
    # the FP32 peak as before; a MUFU-bound one against the least time both pipes together need.
    sysdef = make_system(w["system"])
    _, _, n_exp, gen_ops, gen_mufu, n_pairs = op_counts(sysdef, r["sweep_idx"])
    fma_ops, mufu_ops = L_ALG[w["system"]]
    work, k_bal, alu_pipes = balanced_work(fma_ops, mufu_ops, n_exp, n_pairs)
    dim = sysdef.dim
    rate = per_launch / kern_s   # particle-steps/s of the step kernel
    fma_peak, xu_peak = N_SM * FMA_LANES * f_max, N_SM * XU_LANES * f_max
    cands = {
        "alu": (per_launch * work / kern_s, N_SM * FMA_LANES * f_max,
                "Tops/s (FP32-pipe-equivalent lane-ops of the pipe-balanced work, a*b+c = 1 op)",
                f"148 SM x 128 FP32 lanes x {f_max / 1e6:.0f} MHz (MEASURED_PEAKS sm_max_mhz; FFMA2 / FADD2 / "
                "FMUL2 measured at 126 lane-ops/clk/SM, MUFU 16/clk/SM: profiles/r02_ubench_pipes.txt)", work),
        "hbm": (r["n_local"] * 8 * dim / kern_s, peaks.get("hbm_gbs", 6549.1) * 1e9, "GB/s",
                "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)", 8 * dim / r["S"]),
    }
    if r["image_sum"] > 0 and world == 1:
        # histogram increments: one per binned particle into the L2-resident image (an upper bound on
        # the REDs issued: the warp / block aggregation can only merge them); peak = the measured L2
        # reduction rate on 1-4 M distinct words (profiles/r02_ubench_pipes.txt: 2.14-2.21e11/s)
        cands["l2_red"] = (r["image_sum"] / kern_s, RED_PEAK, "increments/s (1e9)",
                           "measured REDG rate, 4 M distinct words (profiles/r02_ubench_pipes.txt)", 1.0 / r["S"])
    if r["image_sum"] > 0 and world == 1 and r["S"] <= 4:
        # short frames: the state stream and the random-pixel reductions share the L2 and barely overlap
        # (tools/ubench/red_stream.cu: 39 us streaming 201 MB, 51 us for 8.4 M REDs, 75.7 us both in one
        # kernel = 0.84 of the sum). Floor time = 0.84 x (bytes / 5.17 TB/s + increments / 1.64e11/s);
        # reported as a throughput fraction (floor / launch time), "units" = launches.
        t_floor = L2_OVERLAP * (r["n_local"] * 8 * dim / L2_STREAM_BPS + r["image_sum"] / L2_RED_RATE)
        cands["l2_stream_red"] = (1.0 / kern_s, 1.0 / t_floor, "launches/s",
                                  "measured floor of state stream + L2 reductions in one kernel "
                                  "(profiles/r02_ubench_red_stream.txt)", None)
    fracs = {k: v[0] / v[1] for k, v in cands.items()}
    pipe = max(fracs, key=fracs.get)
    ach, peak, unit, src, per_unit = cands[pipe]
    scale = {"alu": 1e12, "l2_stream_red": 1.0}.get(pipe, 1e9)
    roof = {"bound": pipe if pipe != "alu" else "alu", "pipe": alu_pipes if pipe == "alu" else pipe,
            "unit": unit, "achieved": ach / scale,
            "peak": peak / scale, "frac": ach / peak, "peak_source": src,
            "alg_per_particle_step": per_unit,
            "work": {"fma_ops": fma_ops, "mufu_ops": mufu_ops, "exponentials": n_exp, "sigmoid_pairs": n_pairs,
                     "balanced_exponentials_on_fma": k_bal,
                     "generated_fma_ops": gen_ops, "generated_mufu_ops": gen_mufu},
            "fracs_all_pipes": fracs,
            # per pipe: L_alg at the kernel's rate (algorithmic) and the executed op counts (what the
            # pipe actually did; the front end's savings show as algorithmic > executed)
            "pipes": {"fma": {"algorithmic_frac": rate * fma_ops / fma_peak, "executed_frac": rate * gen_ops / fma_peak},
                      "xu": {"algorithmic_frac": rate * mufu_ops / xu_peak, "executed_frac": rate * gen_mufu / xu_peak}},
            "kernel": "ff_step (integrate S steps + project + count, one launch)"}
    roof["traffic"] = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        t = json.load(open(prof)).get(f"{args.config}_S{r['S']}" + ("_noimage" if args.no_image else ""))
        if t:
            roof["traffic"] = t
    if clocks.get("sm_mhz"):
        roof["frac_at_measured_clock"] = roof["frac"] * f_max / (clocks["sm_mhz"] * 1e6)
    line = {"metric": METRIC, "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["t_total_ms"] / args.steps, "higher_is_better": True,
            "scaling": "strong" if w.get("strong") else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (Philox ICs from the paper's IC boxes)", "config": config,
            "pct_fp32_peak": 100 * rate * gen_ops / fma_peak,   # executed FMA-pipe ops (<= 100 by construction)
            "roofline": roof, "clocks": clocks, "gpu_launches": r["launches"], "e2e": r["e2e"],
            "kernel_ms_mean": r["kern_ms"], "frame_ms_p10_p50_p90": [float(np.percentile(r["frame_ms"], q))
                                                                     for q in (10, 50, 90)],
            "image_sum_last_frame": r["image_sum"], "wall_s_timed_region": r["t_wall"],
            "build": __import__("paper_1505_00344_b200.fireflies", fromlist=["x"]).ff_build_info()}
    ctxt = paper_context(w["system"])
    if ctxt:
        line["paper_context"] = ctxt
    if world == 1 and not args.no_cpu_baseline:
        n = reference_sample_size(w, r["S"])
        v, dt, threads, n = cpu_oracle_sample(w, n, r["S"])
        line["cpu_baseline"] = {"value": v, "unit": "particle-steps/s", "cores": threads, "kind": "oracle",
                                "sample": f"{n} particles x {r['S']} RK4 steps + binning ({dt:.1f} s)",
                                "host_cpu": host_cpu_model(),
                                "build": "the scalar oracle as it stands (plain C, gcc -O2 -ffp-contract=off, "
                                         "OpenMP over particles, no SIMD): a correctness reference, not a tuned "
                                         "CPU implementation -- the GPU/CPU ratio is context only",
                                "single_core": single_core_oracle(args.config, max(1024, n // 32), r["S"]),
                                "o3_native": o3_native_oracle(args.config, n, r["S"])}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
