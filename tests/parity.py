"""Shared helpers of the GPU parity tests (test logic only: error metrics and oracle drivers)."""
import numpy as np

import oracle as O


def dim_scales(lo, hi):
    """Per-dimension scale s_d = max |IC box bound|, floored at 1 (parity protocol P2)."""
    return np.maximum(np.maximum(np.abs(np.asarray(lo, np.float64)), np.abs(np.asarray(hi, np.float64))), 1.0)


def scaled_error(gpu, ref, scales):
    """e = |g - o| / max(|o|, s_d) per component; non-finite pairs are handled by finite_mask."""
    g = np.asarray(gpu, np.float64)
    o = np.asarray(ref, np.float64)
    s = np.asarray(scales, np.float64)[:, None]
    return np.abs(g - o) / np.maximum(np.abs(o), s)


def finite_agreement(gpu, ref):
    """Particle is finite in both or non-finite in both (parity protocol non-finite rule)."""
    fg = np.all(np.isfinite(gpu), axis=0)
    fo = np.all(np.isfinite(ref), axis=0)
    return fg == fo, fg & fo


def tier_a(gpu, ref, scales, tol=1e-5):
    same, both = finite_agreement(gpu, ref)
    assert same.all(), f"{(~same).sum()} particles finite on one side only"
    e = scaled_error(gpu[:, both], ref[:, both], scales)
    return float(e.max()) if e.size else 0.0


def oracle_group(model, lo, hi, seed, first, count, params, h, nsteps, sweep_idx=-1, sweep_vals=None):
    """Oracle ICs of a group slice, integrated nsteps in FP32 (the paper's precision)."""
    x = O.ic_uniform(lo, hi, seed, first, count)
    if nsteps:
        x = O.rk4(model, x, np.asarray(params, np.float32), np.float32(h), nsteps, sweep_idx, sweep_vals)
    return x
