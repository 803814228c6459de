"""Full-size parity of the fused image, in the exact launch configuration
bench.py times: the bench's own setup() builds the context (default kernel choice, reset rule,
sweep, camera), one fused frame runs, then the whole state is downloaded and the GPU image must
equal the oracle's histogram of that state bit for bit (the projection and counting are exact
integer / IEEE work, reading R18). The lifted values the oracle bins with are the oracle's own
(O.sweep_values, or O.lifted_values of the GPU's reset counts -- and those must equal what the
library reports). Sampled trajectories of the Lorenz frame are checked against the oracle's
integration and reset rule: redraws bit-exact, kept particles within Tier B."""
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

import oracle as O
from parity import dim_scales, scaled_error

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

ARGS = SimpleNamespace(ppt=0, tpb=0, exchange="nccl", no_image=False, no_reset=False)


def oracle_image(ctx, gids, w, sysdef):
    """The oracle's histogram of the downloaded state of every group (and the lifted values the
    oracle derives for it)."""
    axes, view = bench.projection(w)
    want = np.zeros((w["C"], w["H"], w["W"]), np.uint32)
    for g, (n, _, colour, seed) in zip(gids, w["groups"]):
        x = ctx.read_state(g)
        sv = None
        if "sweep" in w:
            _, a, b, mode, sseed = w["sweep"]
            ep = ctx.read_epochs(g) if "reset" in w else None
            sv = O.lifted_values(a, b, mode, sseed, seed, sysdef.dim, 0, n, n, ep)
            assert np.array_equal(sv.view(np.uint32), ctx.read_lifted(g).view(np.uint32))
        O.histogram(x, axes, view, w["W"], w["H"], w["C"], colour, image=want, sweep_vals=sv)
    return want


# variants of the bench workloads that exercise the other sweep mode with the reset rule
EXTRA = {"sweep_linspace_reset": dict(bench.WORKLOADS["sweep"], sweep=("r", 0.0, 200.0, 1, 5),
                                      reset=(None, None, 0.0)),
         "sweep_philox_reset_bounds": dict(bench.WORKLOADS["sweep"], reset=([-60.0, -80.0, -20.0],
                                                                            [60.0, 80.0, 120.0], 0.0))}


def frame(name, S):
    w = EXTRA.get(name) or bench.WORKLOADS[name]
    ctx, gids, img, _ = bench.setup(ARGS, w, 0, 1)
    img.zero_()
    ctx.step(S, w["dt"])
    ctx.sync()
    return w, ctx, gids, img


@pytest.mark.parametrize("name,S", [("lorenz3d", 100), ("lorenz3d", 10), ("lorenz3d", 1), ("sweep", 100),
                                    ("hh", 100), ("stn_bif3d", 100), ("stn", 1000), ("lorenz3d_collapsed", 100),
                                    ("sweep_linspace_reset", 100), ("sweep_philox_reset_bounds", 100)])
def test_bench_frame_image_is_oracle_histogram_of_its_state(name, S):
    w, ctx, gids, img = frame(name, S)
    sysdef = bench.make_system(w["system"])
    got = ctx.read_image()
    want = oracle_image(ctx, gids, w, sysdef)
    diff = np.count_nonzero(got != want)
    assert diff == 0, f"{diff} pixels differ; sums {int(got.sum())} vs {int(want.sum())}"
    assert int(got.astype(np.int64).sum()) > 0
    if name == "lorenz3d":   # both groups in view: the reset keeps the backward channel populated
        assert got[0].sum() > 0 and got[1].sum() > 0
    # a second frame accumulating into the same image (persistent blocks flush their tables again)
    ctx.step(S, w["dt"])
    ctx.sync()
    want2 = want + oracle_image(ctx, gids, w, sysdef)
    assert np.array_equal(ctx.read_image(), want2)
    ctx.close()


def test_lorenz3d_bench_frame_trajectories_and_resets():
    """configs[1] frame (S = 100, non-finite reset): 2000 sampled particles per group recomputed one by
    one by the oracle -- integration, then the reset rule with the slot's epoch 0. Forward: Tier B of
    100 steps; backward: nearly all blow up and are redrawn -- decisions agree except
    within rounding of the blow-up step, redraws bit-exact; the survivors are only checked finite."""
    w, ctx, gids, img = frame("lorenz3d", 100)
    p = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
    lo, hi = w["box"]
    rng = np.random.default_rng(90)
    for g, (n, d, colour, seed) in zip(gids, w["groups"]):
        idx = np.sort(rng.choice(n, 2000, replace=False))
        got = np.stack([ctx.read_state(g, int(i), 1)[:, 0] for i in idx], axis=1)
        ep = np.array([ctx.read_epochs(g, int(i), 1)[0] for i in idx])
        x0 = np.hstack([O.ic_uniform(lo, hi, seed, int(i), 1) for i in idx])
        want = O.rk4(O.LORENZ, x0, p, np.float32(d * 0.01), 100)
        fin = np.all(np.isfinite(want), axis=0)
        # oracle reset of each sampled particle at its own global index (epoch 0 -> stream 2)
        for j, i in enumerate(idx):
            if not fin[j]:
                col = np.ascontiguousarray(want[:, j:j + 1])
                O.reset(col, None, None, 0.0, 1.0, np.zeros(1, np.float32), np.zeros(1, np.uint32), lo, hi, seed,
                        first_global=int(i))
                want[:, j] = col[:, 0]
        assert np.count_nonzero((ep == 1) != ~fin) <= 4
        red = (ep == 1) & ~fin
        assert np.array_equal(got[:, red].view(np.uint32), want[:, red].view(np.uint32))
        kept = (ep == 0) & fin
        if d > 0:   # Tier B of 100 forward steps (oracle-only proxy: p99 1.1e-5, max 4.6e-4)
            assert kept.sum() == len(idx)
            e = scaled_error(got[:, kept], want[:, kept], dim_scales(lo, hi)).max(axis=0)
            assert np.percentile(e, 99) <= 1e-4 and e.max() <= 1e-2
        else:       # the few backward survivors sit next to a blow-up: no tolerance holds there
            assert red.sum() > 0.9 * len(idx)           # (proxy at 100 steps: p99 5e-2, max 88)
            assert np.all(np.isfinite(got[:, kept]))
    ctx.close()


@pytest.mark.slow
def test_config5_lorenz_1B_frame_image_is_oracle_histogram():
    """configs[4] on one B200 at its full 2^30 particles (12 GB of state), the bench's workload and
    launch (`--config lorenz1b`: non-finite reset, 3-D image): after one fused frame the state is read
    back in 2^26-particle chunks and the oracle's histogram of it, accumulated chunk by chunk, must
    equal the GPU image bit for bit."""
    import os as _os
    try:   # the chunks need ~1 GB of host memory at a time; refuse on a small host rather than swap
        if _os.sysconf("SC_PAGE_SIZE") * _os.sysconf("SC_AVPHYS_PAGES") < (8 << 30):
            pytest.skip("needs >= 8 GB of free host memory")
    except (ValueError, OSError):
        pass
    w, ctx, gids, img = frame("lorenz1b", 100)
    got = ctx.read_image()
    axes, view = bench.projection(w)
    want = np.zeros((w["C"], w["H"], w["W"]), np.uint32)
    (n, _, colour, _), g = w["groups"][0], gids[0]
    chunk = 1 << 26
    for first in range(0, n, chunk):
        O.histogram(ctx.read_state(g, first, min(chunk, n - first)), axes, view, w["W"], w["H"], w["C"], colour,
                    image=want)
    assert np.array_equal(got, want), f"sums {int(got.sum())} vs {int(want.sum())}"
    assert int(want.astype(np.int64).sum()) > n // 4
    ctx.close()


@pytest.mark.parametrize("name", ["lorenz3d", "stn_bif3d", "hh"])
def test_run_to_run_bit_identical(name):
    """Two independent contexts built by the bench's setup() run the same two frames: states, reset
    counts and images are bit-identical (per-particle work is deterministic -- tile scheduling order
    does not touch the arithmetic -- and integer counts commute)."""
    w = bench.WORKLOADS[name]
    runs = []
    for _ in range(2):
        ctx, gids, img, _ = bench.setup(ARGS, w, 0, 1)
        for _ in range(2):
            img.zero_()
            ctx.step(w["S"], w["dt"])
        ctx.sync()
        runs.append(([ctx.read_state(g).view(np.uint32) for g in gids],
                     [ctx.read_epochs(g) if "reset" in w else None for g in gids],
                     img.cpu().numpy().copy()))
        ctx.close()
    (sa, ea, ia), (sb, eb, ib) = runs
    assert all(np.array_equal(a, b) for a, b in zip(sa, sb))
    assert all((a is None and b is None) or np.array_equal(a, b) for a, b in zip(ea, eb))
    assert np.array_equal(ia, ib) and ia.sum() > 0
