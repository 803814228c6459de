"""Oracle-only calibration of the Tier-A parity horizons.

Proxy for "two correct FP32 implementations that differ only by rounding": the FP32 oracle against
the FP64 oracle from the same float32 initial conditions. Calls only oracle/ (no GPU, no product
code). Writes profiles/r02_tier_calibration.json.

  python tools/calibrate_tiers.py [n_particles]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

LO, HI = [-10.0, -30.0, 0.0], [10.0, 30.0, 50.0]   # Fig. 3A box


def scaled_err(a32, b64, scale):
    return np.abs(a32.astype(np.float64) - b64) / np.maximum(np.abs(b64), scale[:, None])


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
    p = np.array([10.0, 28.0, 8.0 / 3.0])
    scale = np.array([10.0, 30.0, 50.0])
    out = {"n_particles": n, "proxy": "oracle FP32 vs oracle FP64, same float32 ICs (Fig. 3A box, seed 3)",
           "cases": []}
    x0 = O.ic_uniform(LO, HI, 3, 0, n)
    for name, h in (("lorenz_r28_forward", 0.01), ("lorenz_r28_backward", -0.01)):
        for steps in (10, 20, 30, 50, 100):
            a = O.rk4(O.LORENZ, x0, p.astype(np.float32), np.float32(h), steps)
            b = O.rk4(O.LORENZ, x0.astype(np.float64), p, float(np.float32(h)), steps)
            fin = np.all(np.isfinite(b), axis=0) & np.all(np.abs(b) < 1e30, axis=0)
            e = scaled_err(a[:, fin], b[:, fin], scale).max(axis=0)
            row = {"case": name, "steps": steps, "finite_fraction": float(fin.mean()),
                   "max": float(e.max()) if e.size else None,
                   "p99": float(np.percentile(e, 99)) if e.size else None,
                   "p99.99": float(np.percentile(e, 99.99)) if e.size else None,
                   "tier_a_holds": bool(e.size and e.max() <= 1e-5)}
            out["cases"].append(row)
            print(row)
    # STN-GPe (reading R6 constants, w_ss = 0), configs[0]: 5k + 5k from (0,1)^2, dt 0.01, 1000 steps
    stn = dict(w_ss=0.0, w_gs=8.971, w_sg=15.168, w_gg=8.502, I=2.216, tau_s=1.0, tau_g=2.77, a_s=2.891,
               theta_s=2.049, a_g=1.826, theta_g=2.032)
    ps = np.array([stn[k] for k in O.PARAMS[O.STN]])
    y0 = O.ic_uniform([0.0, 0.0], [1.0, 1.0], 11, 0, 5000)
    for name, h in (("stn_forward", 0.01), ("stn_backward", -0.01)):
        for steps in (100, 1000):
            a = O.rk4(O.STN, y0, ps.astype(np.float32), np.float32(h), steps)
            b = O.rk4(O.STN, y0.astype(np.float64), ps, float(np.float32(h)), steps)
            e = scaled_err(a, b, np.array([1.0, 1.0])).max(axis=0)
            row = {"case": name, "steps": steps, "finite_fraction": float(np.isfinite(b).all(axis=0).mean()),
                   "max": float(e.max()), "p99": float(np.percentile(e, 99)),
                   "p99.99": float(np.percentile(e, 99.99)), "tier_a_holds": bool(e.max() <= 1e-5)}
            out["cases"].append(row)
            print(row)
    # HH ring N = 3 (readings R7-R11), configs[2]: 2^20 particles in the bench; proxy on n particles
    hh_names = O.hh_param_names(3)
    hh_vals = dict(C=1.0, g_na=120.0, g_k=36.0, g_lk=0.3, e_na=115.0, e_k=-12.0, e_lk=10.613, g_syn=0.5,
                   e_syn=10.0, tau_r=0.5, tau_d=3.0, sigma=5.0, theta=20.0, I1=10.0, I2=10.0, I3=10.0)
    ph = np.array([hh_vals[k] for k in hh_names])
    hlo, hhi = [-20.0, 0, 0, 0, 0] * 3, [100.0, 1, 1, 1, 1] * 3
    hscale = np.maximum(np.maximum(np.abs(np.array(hlo)), np.abs(np.array(hhi))), 1.0)
    z0 = O.ic_uniform(hlo, hhi, 4, 0, min(n, 20000))
    for steps in (10, 30, 100):
        a = O.rk4(O.HH, z0, ph.astype(np.float32), np.float32(0.01), steps)
        b = O.rk4(O.HH, z0.astype(np.float64), ph, float(np.float32(0.01)), steps)
        e = scaled_err(a, b, hscale).max(axis=0)
        row = {"case": "hh_ring3", "steps": steps, "finite_fraction": float(np.isfinite(b).all(axis=0).mean()),
               "max": float(e.max()), "p99": float(np.percentile(e, 99)),
               "p99.99": float(np.percentile(e, 99.99)), "tier_a_holds": bool(e.max() <= 1e-5)}
        out["cases"].append(row)
        print(row)
    # Lorenz with r swept over [0, 200) (Philox, configs[3]), sigma and beta as config 2
    sv = O.sweep_values(0.0, 200.0, 0, 5, 0, n, n)
    x0s = O.ic_uniform(LO, HI, 5, 0, n)
    ps = np.array([10.0, 0.0, 8.0 / 3.0])
    for steps in (10, 30):
        a = O.rk4(O.LORENZ, x0s, ps.astype(np.float32), np.float32(0.01), steps, 1, sv)
        b = O.rk4(O.LORENZ, x0s.astype(np.float64), ps, float(np.float32(0.01)), steps, 1, sv.astype(np.float64))
        e = scaled_err(a, b, scale).max(axis=0)
        row = {"case": "lorenz_swept_r", "steps": steps, "finite_fraction": 1.0, "max": float(e.max()),
               "p99": float(np.percentile(e, 99)), "p99.99": float(np.percentile(e, 99.99)),
               "tier_a_holds": bool(e.max() <= 1e-5)}
        out["cases"].append(row)
        print(row)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", "r02_tier_calibration.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
