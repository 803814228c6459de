"""Measure GPU-vs-oracle scaled-error percentiles per workload and horizon (calibration data for the
parity tiers in DESIGN.md; run on the GPU box). Prints one JSON object per (case, steps)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
import paper_1505_00344_b200 as FF  # noqa: E402
from paper_1505_00344_b200 import systems  # noqa: E402
from parity import dim_scales, finite_agreement, scaled_error  # noqa: E402


def stats(tag, steps, got, want, sc):
    same, both = finite_agreement(got, want)
    e = scaled_error(got[:, both], want[:, both], sc).max(axis=0)
    out = {"case": tag, "steps": steps, "n": int(got.shape[1]), "finite_mismatch": int((~same).sum()),
           "nonfinite": int((~both).sum())}
    for q in (50, 99, 99.9, 99.99):
        out[f"p{q}"] = float(np.percentile(e, q)) if e.size else None
    out["max"] = float(e.max()) if e.size else None
    print(json.dumps(out), flush=True)


def run(tag, sysdef, model, lo, hi, n, params, direction, checkpoints, ppt=0, sweep=None, set_params=None):
    ctx = FF.Context(sysdef, [n])
    if ppt:
        ctx.set_launch(ppt, 256 if ppt == 1 else 128)
    for k, v in (set_params or {}).items():
        ctx.set_param(k, v)
    g = ctx.init_group(lo, hi, n, direction, 0, seed=7)
    sidx, sv = -1, None
    if sweep:
        name, a, b = sweep
        ctx.sweep_param(g, name, a, b, 0, 5)
        sidx = [p[0] for p in sysdef.params].index(name)
        sv = O.sweep_values(a, b, 0, 5, 0, n, n)
    x = O.ic_uniform(lo, hi, 7, 0, n)
    done = 0
    sc = dim_scales(lo, hi)
    h = np.float32(0.01 * direction)
    for c in checkpoints:
        ctx.step(c - done, 0.01)
        x = O.rk4(model, x, params, h, c - done, sidx, sv)
        done = c
        stats(f"{tag}/ppt{ppt}", c, ctx.read_state(g), x, sc)
    ctx.close()


def main():
    lz = systems.lorenz()
    LZ_LO, LZ_HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]
    p28 = np.array([10.0, 28.0, 8.0 / 3.0], np.float32)
    for ppt in (1, 2):
        run("lorenz28_fwd", lz, O.LORENZ, LZ_LO, LZ_HI, 100000, p28, 1, [10, 30, 50, 100, 300], ppt)
        run("lorenz28_bwd", lz, O.LORENZ, LZ_LO, LZ_HI, 100000, p28, -1, [5, 10, 20, 30, 50], ppt)
        run("lorenz_sweep", lz, O.LORENZ, LZ_LO, LZ_HI, 100000, p28, 1, [5, 10, 50, 100], ppt, sweep=("r", 0.0, 200.0))
        st = systems.stn_gpe()
        ps = np.array([p[1] for p in st.params], np.float32)
        run("stn_fwd", st, O.STN, [0, 0], [1, 1], 50000, ps, 1, [100, 1000], ppt)
        run("stn_bwd", st, O.STN, [0, 0], [1, 1], 50000, ps, -1, [100, 1000], ppt)
        hh = systems.hh_ring(3)
        d = {p[0]: p[1] for p in hh.params}
        ph = np.array([d[k] for k in O.hh_param_names(3)], np.float32)
        run("hh3", hh, O.HH, [-20.0, 0, 0, 0, 0] * 3, [100.0, 1, 1, 1, 1] * 3, 20000, ph, 1, [10, 100, 1000], ppt)
    # the default (bench) launch at a size that selects the pipe-balanced kernel (FMA-pipe reciprocals)
    st = systems.stn_gpe()
    ps = np.array([p[1] for p in st.params], np.float32)
    run("stn_bif_fwd", st, O.STN, [0, 0], [1, 1], 100000, ps, 1, [100, 1000], 0, sweep=("w_ss", 0.0, 12.0))
    run("stn_bif_bwd", st, O.STN, [0, 0], [1, 1], 100000, ps, -1, [100], 0, sweep=("w_ss", 0.0, 12.0))


if __name__ == "__main__":
    main()
